// nacs_warp.cu — warp-per-request TOPSIS batch kernel (nacs_schedule_batch fast path).
//
// Every warp schedules whole requests on its own (no block barrier anywhere): all warps
// of a CTA share one read-only copy of the snapshot in shared memory (criteria table as
// padded int32 SoA, fabric links as u16), and each warp keeps a private *overlay* of
// the servers and links its current request has modified (R21 snapshot isolation).
// Scans of the n servers go 128 servers per warp iteration (4 consecutive servers per
// lane, int4 loads); the few servers that are special in a pod step (overlaid, excluded
// or flow endpoints) are merged into the scan through a sorted list.  Fabric-table rows
// (edge-agg rows, agg-core rows) touched by the overlay are flagged dirty and read
// through the overlay; clean rows are read straight from the snapshot.
//
// Requests beyond the fast-path limits (containers > 32, vlinks > 64, or overlay /
// exclusion overflow) are appended to a deferred list that the CTA-per-request kernel
// (nacs_kernels.cu, k_batch) schedules afterwards; both produce identical results.
//
// The method steps and readings are those of nacs_kernels.cu.
#include "nacs_device.cuh"

namespace nacs {

namespace {
constexpr int WC = 32;    // containers per request (fast path)
constexpr int WV = 64;    // vlinks per request
constexpr int WOS = 32;   // overlay servers
constexpr int WOL = 128;  // overlay fabric links
constexpr int WSP = 64;   // specials per pod step
constexpr int WF = 32;    // flows per pod step
constexpr int WX = 32;    // exclusions per pod step
constexpr int WLOG = 256; // undo-log entries per commit
}  // namespace

struct WScr {
  int nos, nol, nflow, sumD, G, nsp, nex, pad0;
  int os_u[WOS], os_cpu[WOS], os_ram[WOS], os_act[WOS], os_acc[WOS];
  int ol_id[WOL], ol_val[WOL];
  int pod_srv[WC];
  int fv[WF], fD[WF], fok[WF], fpath[WF];
  int sp_u[WSP], sp_info[WSP];
  int ex[WX];
  // dynamic tail: dirty[(E + k*h + 31)/32] | edgebad[(E+31)/32] | pm[k]
};

template <typename LT>
struct WCtx {
  int k, h, n, npad, E, nfabea;  // nfabea = E*h (start of agg-core links in fab[])
  unsigned magic;
  const int4 *cpu4, *ram4, *act4, *acc4;  // criteria SoA (shared)
  const int *cpu, *ram, *act, *acc;
  const LT* fab;                           // edge-agg[E*h] | agg-core[k*h*h] (shared)
  WScr* w;
  unsigned *dirty, *edgebad, *pm;
  int4* ulog;
  int ulog_n;
  int lane;
  Opt o;
};

// ------------------------------------------------------------ overlay reads --
// fabric link fid (per lane): overlay value if its row is dirty and it is overlaid
template <typename LT>
__device__ __forceinline__ int fab_val(const WCtx<LT>& c, int fid) {
  int v = (int)c.fab[fid];
  unsigned row = div_h((unsigned)fid, c.magic);
  if ((c.dirty[row >> 5] >> (row & 31)) & 1u) {
    const WScr* w = c.w;
    for (int s = 0; s < w->nol; ++s)
      if (w->ol_id[s] == fid) v = w->ol_val[s];
  }
  return v;
}
template <typename LT>
__device__ __forceinline__ bool row_dirty(const WCtx<LT>& c, int row) {
  return (c.dirty[row >> 5] >> (row & 31)) & 1u;
}
// overlay slot of server u, -1 if none (per lane)
template <typename LT>
__device__ __forceinline__ int os_slot(const WCtx<LT>& c, int u) {
  const WScr* w = c.w;
  int s = -1;
  for (int i = 0; i < w->nos; ++i)
    if (w->os_u[i] == u) s = i;
  return s;
}
template <typename LT>
__device__ __forceinline__ int acc_val(const WCtx<LT>& c, int u) {
  int s = os_slot(c, u);
  return s >= 0 ? c.w->os_acc[s] : c.acc[u];
}

// ----------------------------------------------------- overlay writes (lane 0) --
// returns false on overflow
template <typename LT>
__device__ bool set_server(WCtx<LT>& c, int u, int cpu, int ram, int act, int acc, bool log = true) {
  WScr* w = c.w;
  int s = os_slot(c, u);
  if (s < 0) {
    if (w->nos >= WOS) return false;
    s = w->nos++;
    w->os_u[s] = u;
  } else if (!log) {
  } else if (c.ulog_n < WLOG) {
    c.ulog[c.ulog_n++] = make_int4(s, w->os_cpu[s], w->os_ram[s], w->os_acc[s] * 2 + w->os_act[s]);
  } else {
    return false;
  }
  w->os_cpu[s] = cpu;
  w->os_ram[s] = ram;
  w->os_act[s] = act;
  w->os_acc[s] = acc;
  return true;
}
template <typename LT>
__device__ bool set_link(WCtx<LT>& c, int fid, int val, bool log = true) {
  WScr* w = c.w;
  int s = -1;
  for (int i = 0; i < w->nol; ++i)
    if (w->ol_id[i] == fid) s = i;
  if (s < 0) {
    if (w->nol >= WOL) return false;
    s = w->nol++;
    w->ol_id[s] = fid;
  } else if (!log) {
  } else if (c.ulog_n < WLOG) {
    c.ulog[c.ulog_n++] = make_int4(-1 - s, w->ol_val[s], 0, 0);
  } else {
    return false;
  }
  w->ol_val[s] = val;
  unsigned row = div_h((unsigned)fid, c.magic);
  c.dirty[row >> 5] |= 1u << (row & 31);
  return true;
}
template <typename LT>
__device__ void undo_commit(WCtx<LT>& c, int nos0, int nol0) {
  WScr* w = c.w;
  for (int i = c.ulog_n - 1; i >= 0; --i) {
    int4 e = c.ulog[i];
    if (e.x >= 0) {
      w->os_cpu[e.x] = e.y;
      w->os_ram[e.x] = e.z;
      w->os_acc[e.x] = e.w >> 1;
      w->os_act[e.x] = e.w & 1;
    } else {
      w->ol_val[-1 - e.x] = e.y;
    }
  }
  w->nos = nos0;
  w->nol = nol0;
  c.ulog_n = 0;
}

// fabric link ids of path pid between servers u, v (same numbering as fab[])
template <typename LT>
__device__ __forceinline__ int path_fids(const WCtx<LT>& c, int u, int v, int pid, int fid[4]) {
  if (pid <= 0) return 0;
  int h = c.h;
  int eu = (int)div_h(u, c.magic), ev = (int)div_h(v, c.magic);
  if (pid <= h) {
    int a = pid - 1;
    fid[0] = eu * h + a;
    fid[1] = ev * h + a;
    return 2;
  }
  int t = pid - 1 - h;
  int a = (int)div_h(t, c.magic), b = t - a * h;
  int pu = (int)div_h(eu, c.magic), pv = (int)div_h(ev, c.magic);
  fid[0] = eu * h + a;
  fid[1] = c.nfabea + (pu * h + a) * h + b;
  fid[2] = c.nfabea + (pv * h + a) * h + b;
  fid[3] = ev * h + a;
  return 4;
}

// R16: widest ECMP path u -> v on current residuals (snapshot + overlay); warp-wide.
template <typename LT>
__device__ int2 wpath(const WCtx<LT>& c, int u, int v) {
  int h = c.h;
  int eu = (int)div_h(u, c.magic), ev = (int)div_h(v, c.magic);
  if (eu == ev) return make_int2(0, INT_MAX);
  int pu = (int)div_h(eu, c.magic), pv = (int)div_h(ev, c.magic);
  int best = -1, bt = INT_MAX;
  if (pu == pv) {
    for (int a = c.lane; a < h; a += 32) {
      int b = min(fab_val(c, eu * h + a), fab_val(c, ev * h + a));
      if (b > best) { best = b; bt = a; }
    }
  } else {
    for (int t = c.lane; t < h * h; t += 32) {
      int a = (int)div_h(t, c.magic), b = t - a * h;
      int x = min(min(fab_val(c, eu * h + a), fab_val(c, ev * h + a)),
                  min(fab_val(c, c.nfabea + (pu * h + a) * h + b), fab_val(c, c.nfabea + (pv * h + a) * h + b)));
      if (x > best) { best = x; bt = t; }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    int ob = __shfl_xor_sync(NACS_FULL, best, o);
    int ot = __shfl_xor_sync(NACS_FULL, bt, o);
    if (ob > best || (ob == best && ot < bt)) { best = ob; bt = ot; }
  }
  return make_int2(pu == pv ? 1 + bt : 1 + h + bt, best);
}

// a2: edge switches some flow cannot reach with its demand (threshold bitmasks).
template <typename LT>
__device__ void wfabric(WCtx<LT>& c) {
  WScr* w = c.w;
  const int h = c.h, k = c.k, E = c.E;
  const int nEW = (E + 31) >> 5;
  for (int i = c.lane; i < nEW; i += 32) c.edgebad[i] = 0u;
  for (int f = 0; f < w->nflow; ++f) {
    const int v = w->fv[f], D = w->fD[f];
    const int ev = (int)div_h(v, c.magic), pv = (int)div_h(ev, c.magic);
    for (int p = c.lane; p < k; p += 32) c.pm[p] = 0u;
    // vb: core columns b reachable from pod pv through aggregation a (lane a)
    unsigned vb = 0;
    bool vme = false;
    if (c.lane < h) {
      int a = c.lane;
      int row = E + pv * h + a;
      const LT* r = c.fab + c.nfabea + (pv * h + a) * h;
      if (!row_dirty(c, row)) {
        for (int b = 0; b < h; ++b) vb |= ((int)r[b] >= D ? 1u : 0u) << b;
      } else {
        for (int b = 0; b < h; ++b) vb |= (fab_val(c, c.nfabea + (pv * h + a) * h + b) >= D ? 1u : 0u) << b;
      }
      vme = fab_val(c, ev * h + a) >= D;
    }
    const unsigned vm = __ballot_sync(NACS_FULL, vme);
    __syncwarp();
    // pm[p] bit a: some core (a, b) joins pod p and pod pv with both links >= D
    const int items = k * h;
    for (int t0 = 0; t0 < items; t0 += 32) {
      int t = t0 + c.lane;
      int p = 0, a = 0;
      bool ok = false;
      if (t < items) {
        p = (int)div_h(t, c.magic);
        a = t - p * h;
      }
      unsigned vba = __shfl_sync(NACS_FULL, vb, a);
      if (t < items && ((vm >> a) & 1u)) {
        unsigned bits = 0;
        int row = E + p * h + a;
        const LT* r = c.fab + c.nfabea + (p * h + a) * h;
        if (!row_dirty(c, row)) {
          for (int b = 0; b < h; ++b) bits |= ((int)r[b] >= D ? 1u : 0u) << b;
        } else {
          for (int b = 0; b < h; ++b) bits |= (fab_val(c, c.nfabea + (p * h + a) * h + b) >= D ? 1u : 0u) << b;
        }
        ok = (bits & vba) != 0u;
      }
      if (ok) atomicOr(&c.pm[p], 1u << a);
    }
    __syncwarp();
    for (int e0 = 0; e0 < E; e0 += 32) {
      int e = e0 + c.lane;
      bool bad = false;
      if (e < E && e != ev) {
        unsigned em = 0;
        if (!row_dirty(c, e)) {
          const LT* r = c.fab + e * h;
          for (int a = 0; a < h; ++a) em |= ((int)r[a] >= D ? 1u : 0u) << a;
        } else {
          for (int a = 0; a < h; ++a) em |= (fab_val(c, e * h + a) >= D ? 1u : 0u) << a;
        }
        int pe = (int)div_h(e, c.magic);
        unsigned ok = (pe == pv) ? (em & vm) : (em & vm & c.pm[pe]);
        bad = ok == 0u;
      }
      unsigned bw = __ballot_sync(NACS_FULL, bad);
      if (c.lane == 0) c.edgebad[e0 >> 5] |= bw;
    }
    __syncwarp();
  }
}

// Criteria of 4 consecutive servers (lane) with the pod step's special servers merged in.
struct Four {
  int4 c, r, a, q;
  int info[4];  // 0 = ordinary, else special info word
};

__device__ __forceinline__ void set_comp(int4& v, int j, int x) {
  if (j == 0) v.x = x;
  else if (j == 1) v.y = x;
  else if (j == 2) v.z = x;
  else v.w = x;
}
__device__ __forceinline__ int get_comp(const int4& v, int j) {
  return j == 0 ? v.x : (j == 1 ? v.y : (j == 2 ? v.z : v.w));
}

template <typename LT>
__device__ __forceinline__ void load_four(const WCtx<LT>& c, int chunk, int base, int& sp_ptr, Four& f) {
  const int li = chunk * 32 + c.lane;
  f.c = c.cpu4[li];
  f.r = c.ram4[li];
  f.a = c.act4[li];
  f.q = c.acc4[li];
  f.info[0] = f.info[1] = f.info[2] = f.info[3] = 0;
  const WScr* w = c.w;
  if (sp_ptr < w->nsp && w->sp_u[sp_ptr] < base + 128) {
    while (sp_ptr < w->nsp && w->sp_u[sp_ptr] < base + 128) {
      int u = w->sp_u[sp_ptr], info = w->sp_info[sp_ptr];
      if (((u - base) >> 2) == c.lane) {
        int j = (u - base) & 3;
        int slot = (info & 63) - 1;
        if (slot >= 0) {
          set_comp(f.c, j, w->os_cpu[slot]);
          set_comp(f.r, j, w->os_ram[slot]);
          set_comp(f.a, j, w->os_act[slot]);
          set_comp(f.q, j, w->os_acc[slot]);
        }
        f.info[j] = info;
      }
      ++sp_ptr;
    }
  }
}

struct StepP {
  int dc, dr, sumD;
  bool net, G, pf;
};

// a3: feasibility of server u with criteria (x0, x1, x3) and special info
template <typename LT>
__device__ __forceinline__ bool feasible(const WCtx<LT>& c, const StepP& sp, int u, int x0, int x1, int x3,
                                         int info) {
  bool ok = x0 >= sp.dc && x1 >= sp.dr;
  if (info == 0) {
    if (sp.net) {
      unsigned e = div_h((unsigned)u, c.magic);
      ok = ok && sp.G && x3 >= sp.sumD && !((c.edgebad[e >> 5] >> (e & 31)) & 1u);
    }
    return ok;
  }
  if (info & 64) return false;  // excluded (R18)
  int f = (info >> 7) - 1;
  if (f >= 0) return ok && (!sp.pf || c.w->fok[f]);  // its own flow needs no network
  if (sp.net) {
    unsigned e = div_h((unsigned)u, c.magic);
    ok = ok && sp.G && x3 >= sp.sumD && !((c.edgebad[e >> 5] >> (e & 31)) & 1u);
  }
  return ok;
}

// Build the sorted special list: overlay servers, excluded servers, flow servers.
template <typename LT>
__device__ void build_specials(WCtx<LT>& c) {
  WScr* w = c.w;
  const int l = c.lane;
  // entry A: overlay slot l; entry B: excluded server l not in the overlay
  bool va = l < w->nos, vbx = false;
  int ua = va ? w->os_u[l] : INT_MAX, ia = 0;
  if (va) {
    bool ex = false;
    for (int i = 0; i < w->nex; ++i) ex |= w->ex[i] == ua;
    int f = -1;
    for (int i = 0; i < w->nflow; ++i)
      if (w->fv[i] == ua) f = i;
    ia = (l + 1) | (ex ? 64 : 0) | ((f + 1) << 7);
  }
  int ub = INT_MAX;
  if (l < w->nex) {
    ub = w->ex[l];
    vbx = os_slot(c, ub) < 0;
    if (!vbx) ub = INT_MAX;
  }
  int ra = 0, rb = 0;
  for (int s = 0; s < 32; ++s) {
    int xa = __shfl_sync(NACS_FULL, ua, s);
    int xb = __shfl_sync(NACS_FULL, ub, s);
    ra += (xa < ua) + (xb < ua);
    rb += (xa < ub) + (xb < ub);
  }
  if (va) { w->sp_u[ra] = ua; w->sp_info[ra] = ia; }
  if (vbx) { w->sp_u[rb] = ub; w->sp_info[rb] = 64; }
  int cnt = __popc(__ballot_sync(NACS_FULL, va)) + __popc(__ballot_sync(NACS_FULL, vbx));
  if (l == 0) w->nsp = cnt;
  __syncwarp();
}

struct WStats {
  unsigned long long steps, retries, fp64, invalid, feas;
};

template <typename LT>
__global__ void __launch_bounds__(512, 1) k_batch_warp(Geo g, Opt o, const int* __restrict__ state, ReqsDev R,
                                                       OutDev O, int4* ulog_all, int* next, int* deferred,
                                                       int* n_deferred, unsigned long long* stats) {
  extern __shared__ __align__(16) unsigned char dyn[];
  const int n = g.n, h = g.h, k = g.k, E = g.E;
  const int npad = (n + 127) & ~127;
  // ---- a0: shared snapshot (read-only for the whole kernel)
  int* scpu = reinterpret_cast<int*>(dyn);
  int* sram = scpu + npad;
  int* sact = sram + npad;
  int* sacc = sact + npad;
  LT* sfab = reinterpret_cast<LT*>(sacc + npad);
  const int nfab = E * h + k * h * h;
  size_t off = (size_t)16 * npad + (((size_t)sizeof(LT) * nfab + 15) & ~(size_t)15);
  const int nDW = (E + k * h + 31) >> 5, nEW = (E + 31) >> 5;
  const size_t wbytes = ((sizeof(WScr) + 4 * (nDW + nEW + k)) + 15) & ~(size_t)15;
  for (int i = threadIdx.x; i < npad; i += blockDim.x) {
    bool in = i < n;
    scpu[i] = in ? state[i] : -1;  // padding is never feasible (demands are > 0)
    sram[i] = in ? state[n + i] : -1;
    sact[i] = in ? state[2 * n + i] : 0;
    sacc[i] = in ? state[3 * n + i] : 0;
  }
  for (int i = threadIdx.x; i < nfab; i += blockDim.x) sfab[i] = (LT)state[4 * n + i];
  __syncthreads();  // the only block barrier: the snapshot is complete

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  WCtx<LT> c;
  c.k = k; c.h = h; c.n = n; c.npad = npad; c.E = E; c.nfabea = E * h;
  c.magic = g.magic_h;
  c.cpu = scpu; c.ram = sram; c.act = sact; c.acc = sacc;
  c.cpu4 = reinterpret_cast<const int4*>(scpu);
  c.ram4 = reinterpret_cast<const int4*>(sram);
  c.act4 = reinterpret_cast<const int4*>(sact);
  c.acc4 = reinterpret_cast<const int4*>(sacc);
  c.fab = sfab;
  unsigned char* wb = dyn + off + (size_t)warp * wbytes;
  c.w = reinterpret_cast<WScr*>(wb);
  c.dirty = reinterpret_cast<unsigned*>(wb + sizeof(WScr));
  c.edgebad = c.dirty + nDW;
  c.pm = c.edgebad + nEW;
  c.ulog = ulog_all + ((size_t)blockIdx.x * (blockDim.x >> 5) + warp) * WLOG;
  c.ulog_n = 0;
  c.lane = lane;
  c.o = o;
  WScr* w = c.w;
  for (int i = lane; i < nDW; i += 32) c.dirty[i] = 0u;
  if (lane == 0) { w->nos = 0; w->nol = 0; }
  __syncwarp();
  const int nchunks = npad >> 7;
  const bool h4 = (h & 3) == 0;
  WStats ws = {0, 0, 0, 0, 0};
  double wd[4] = {o.wd[0], o.wd[1], o.wd[2], o.wd[3]};

  for (;;) {
    int r = 0;
    if (lane == 0) r = atomicAdd(next, 1);
    r = __shfl_sync(NACS_FULL, r, 0);
    if (r >= R.n) break;
    const int c0 = R.coff[r], nC = R.coff[r + 1] - c0;
    const int v0 = R.voff[r], nV = R.voff[r + 1] - v0;
    if (nC > WC || nV > WV || nC <= 0 || nV < 0) {
      if (nC > WC || nV > WV) {
        if (lane == 0) deferred[atomicAdd(n_deferred, 1)] = r;
        continue;
      }
    }
    // request registers: container `lane`, vlinks `lane` and `lane + 32`
    const bool hc = lane < nC;
    int cmin = 1, cmax = 1, rmin = 1, rmax = 1, cpod = 0;
    if (hc) {
      cmin = R.cpu_min[c0 + lane]; cmax = R.cpu_max[c0 + lane];
      rmin = R.ram_min[c0 + lane]; rmax = R.ram_max[c0 + lane];
      cpod = R.pod_of[c0 + lane];
    }
    const bool hv0 = lane < nV, hv1 = lane + 32 < nV;
    int s0 = 0, d0 = 1, bn0 = 1, bx0 = 1, s1 = 0, d1 = 1, bn1 = 1, bx1 = 1;
    if (hv0) { s0 = R.src[v0 + lane]; d0 = R.dst[v0 + lane]; bn0 = R.bw_min[v0 + lane]; bx0 = R.bw_max[v0 + lane]; }
    if (hv1) { s1 = R.src[v0 + lane + 32]; d1 = R.dst[v0 + lane + 32]; bn1 = R.bw_min[v0 + lane + 32]; bx1 = R.bw_max[v0 + lane + 32]; }
    // validation (R24), all in registers
    bool bad = hc && (cmin <= 0 || rmin <= 0 || cmin > cmax || rmin > rmax || cpod < 0 || cpod >= nC);
    bad |= hv0 && (s0 < 0 || s0 >= nC || d0 < 0 || d0 >= nC || s0 == d0 || bn0 <= 0 || bn0 > bx0);
    bad |= hv1 && (s1 < 0 || s1 >= nC || d1 < 0 || d1 >= nC || s1 == d1 || bn1 <= 0 || bn1 > bx1);
    unsigned used = __reduce_or_sync(NACS_FULL, hc && cpod >= 0 && cpod < 32 ? (1u << cpod) : 0u);
    int maxp = (int)__reduce_max_sync(NACS_FULL, hc && cpod >= 0 ? (unsigned)cpod : 0u);
    bool invalid = __any_sync(NACS_FULL, bad) || nC <= 0 || maxp >= 32 ||
                   used != (maxp == 31 ? 0xffffffffu : ((1u << (maxp + 1)) - 1u));
    if (invalid) {
      if (hc) { O.server[c0 + lane] = -1; O.cpu_a[c0 + lane] = 0; O.ram_a[c0 + lane] = 0; }
      if (hv0) { O.bw_a[v0 + lane] = 0; O.path[v0 + lane] = -1; }
      if (hv1) { O.bw_a[v0 + lane + 32] = 0; O.path[v0 + lane + 32] = -1; }
      if (lane == 0) { O.status[r] = -1; ws.invalid += 1; }
      continue;
    }
    const int P = maxp + 1;
    // pod demands (lane p): sum of c^min over the pod's containers
    int pcpu = 0, pram = 0;
    for (int i = 0; i < nC; ++i) {
      int pd = __shfl_sync(NACS_FULL, cpod, i);
      int cm = __shfl_sync(NACS_FULL, cmin, i);
      int rm = __shfl_sync(NACS_FULL, rmin, i);
      if (lane == pd) { pcpu += cm; pram += rm; }
    }
    // pods of the vlink endpoints
    const int pa0 = __shfl_sync(NACS_FULL, cpod, s0 & 31), pb0 = __shfl_sync(NACS_FULL, cpod, d0 & 31);
    const int pa1 = __shfl_sync(NACS_FULL, cpod, s1 & 31), pb1 = __shfl_sync(NACS_FULL, cpod, d1 & 31);
    int path0 = -1, path1 = -1;
    w->pod_srv[lane] = -1;
    if (lane == 0) { w->nos = 0; w->nol = 0; }
    __syncwarp();
    bool rejected = false, defer = false;

    for (int p = 0; p < P && !rejected && !defer; ++p) {
      // ---- a1/a2: flows of pod p to placed peers, aggregated per server (R17)
      int ov0 = -1, ov1 = -1;
      if (hv0) {
        int other = (pa0 == p && pb0 != p) ? pb0 : ((pb0 == p && pa0 != p) ? pa0 : -1);
        if (other >= 0) ov0 = w->pod_srv[other];
      }
      if (hv1) {
        int other = (pa1 == p && pb1 != p) ? pb1 : ((pb1 == p && pa1 != p) ? pa1 : -1);
        if (other >= 0) ov1 = w->pod_srv[other];
      }
      bool has0 = ov0 >= 0, has1 = ov1 >= 0;
      if (lane == 0) { w->nflow = 0; w->nex = 0; }
      __syncwarp();
      int sumD = 0;
      for (;;) {
        unsigned m0 = __ballot_sync(NACS_FULL, has0), m1 = __ballot_sync(NACS_FULL, has1);
        if (!(m0 | m1)) break;
        int src_l = m0 ? __ffs(m0) - 1 : __ffs(m1) - 1;
        int cand = m0 ? ov0 : ov1;
        int vsel = __shfl_sync(NACS_FULL, cand, src_l);
        bool mine0 = has0 && ov0 == vsel, mine1 = has1 && ov1 == vsel;
        int D = (int)__reduce_add_sync(NACS_FULL, (mine0 ? (unsigned)bn0 : 0u) + (mine1 ? (unsigned)bn1 : 0u));
        has0 &= !mine0;
        has1 &= !mine1;
        sumD += D;
        if (lane == 0) {  // insert sorted by server
          int nf = w->nflow, i = nf;
          while (i > 0 && w->fv[i - 1] > vsel) { w->fv[i] = w->fv[i - 1]; w->fD[i] = w->fD[i - 1]; --i; }
          w->fv[i] = vsel;
          w->fD[i] = D;
          w->nflow = nf + 1;
        }
        __syncwarp();
      }
      const int nflow = w->nflow;
      const bool net = o.path_filter && nflow > 0;
      if (net) wfabric(c);
      // fok (lane f) and G
      bool Gl = true;
      if (lane < nflow) {
        int v = w->fv[lane], D = w->fD[lane];
        int av = acc_val(c, v);
        Gl = av >= D;
        bool fk = av >= sumD - D;
        for (int f2 = 0; f2 < nflow; ++f2)
          if (f2 != lane && acc_val(c, w->fv[f2]) < w->fD[f2]) fk = false;
        if (net) {
          unsigned e = div_h((unsigned)v, c.magic);
          if ((c.edgebad[e >> 5] >> (e & 31)) & 1u) fk = false;
        }
        w->fok[lane] = fk;
      }
      const bool G = __all_sync(NACS_FULL, Gl);
      const int dc = __shfl_sync(NACS_FULL, pcpu, p), dr = __shfl_sync(NACS_FULL, pram, p);
      StepP sp{dc, dr, sumD, net, G, o.path_filter != 0};
      __syncwarp();

      for (;;) {  // attempts of this pod step (R18 retries)
        build_specials(c);
        // ---- a3 + a4: filter and statistics
        int nf = 0, nact = 0;
        unsigned mn0 = UINT_MAX, mn1 = UINT_MAX, mn3 = UINT_MAX, mx0 = 0, mx1 = 0, mx3 = 0;
        unsigned long long q0 = 0, q1 = 0, q3 = 0;
        int spp = 0;
        for (int ch = 0; ch < nchunks; ++ch) {
          const int base = ch << 7;
          Four f;
          load_four(c, ch, base, spp, f);
          const int u0 = base + 4 * lane;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            int x0 = get_comp(f.c, j), x1 = get_comp(f.r, j), x2 = get_comp(f.a, j), x3 = get_comp(f.q, j);
            bool ok = feasible(c, sp, u0 + j, x0, x1, x3, f.info[j]);
            if (ok) {
              nf += 1;
              nact += x2;
              mn0 = min(mn0, (unsigned)x0); mx0 = max(mx0, (unsigned)x0);
              mn1 = min(mn1, (unsigned)x1); mx1 = max(mx1, (unsigned)x1);
              mn3 = min(mn3, (unsigned)x3); mx3 = max(mx3, (unsigned)x3);
              q0 += (unsigned long long)(unsigned)x0 * (unsigned)x0;
              q1 += (unsigned long long)(unsigned)x1 * (unsigned)x1;
              q3 += (unsigned long long)(unsigned)x3 * (unsigned)x3;
            }
          }
        }
        (void)h4;
        nf = (int)__reduce_add_sync(NACS_FULL, (unsigned)nf);
        ws.steps += 1;
        ws.feas += (unsigned long long)nf;
        if (nf == 0) { rejected = true; break; }  // R20
        nact = (int)__reduce_add_sync(NACS_FULL, (unsigned)nact);
        TopsisP tp;
        tp.mn[0] = (int)__reduce_min_sync(NACS_FULL, mn0); tp.mx[0] = (int)__reduce_max_sync(NACS_FULL, mx0);
        tp.mn[1] = (int)__reduce_min_sync(NACS_FULL, mn1); tp.mx[1] = (int)__reduce_max_sync(NACS_FULL, mx1);
        tp.mn[3] = (int)__reduce_min_sync(NACS_FULL, mn3); tp.mx[3] = (int)__reduce_max_sync(NACS_FULL, mx3);
        tp.mn[2] = nact == nf ? 1 : 0;
        tp.mx[2] = nact > 0 ? 1 : 0;
        unsigned long long sq[4] = {warp_sum_u64(q0), warp_sum_u64(q1), (unsigned long long)nact, warp_sum_u64(q3)};
        topsis_params(tp, wd, sq);
        // ---- a5T + a7: closeness and top-2 argmax key
        unsigned long long k1 = 0, k2 = 0;
        spp = 0;
        for (int ch = 0; ch < nchunks; ++ch) {
          const int base = ch << 7;
          Four f;
          load_four(c, ch, base, spp, f);
          const int u0 = base + 4 * lane;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            int x0 = get_comp(f.c, j), x1 = get_comp(f.r, j), x2 = get_comp(f.a, j), x3 = get_comp(f.q, j);
            if (feasible(c, sp, u0 + j, x0, x1, x3, f.info[j])) {
              float rr = topsis32(tp, x0, x1, x2, x3);
              top2_insert(k1, k2, score_key(rr, u0 + j));
            }
          }
        }
        warp_top2(k1, k2);
        int best = (int)(0xFFFFFFFFu - (unsigned)(k1 & 0xFFFFFFFFull));
        const float s1 = __uint_as_float((unsigned)(k1 >> 32)), s2 = __uint_as_float((unsigned)(k2 >> 32));
        if (o.exact64 || (k2 != 0ull && s1 - s2 <= kTopsisDelta)) {  // R14: FP64 near-tie re-decision
          const float thr = o.exact64 ? -1.0f : s1 - 2.0f * kTopsisDelta;
          double bv = -DBL_MAX;
          int bj = -1;
          spp = 0;
          for (int ch = 0; ch < nchunks; ++ch) {
            const int base = ch << 7;
            Four f;
            load_four(c, ch, base, spp, f);
            const int u0 = base + 4 * lane;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              int x0 = get_comp(f.c, j), x1 = get_comp(f.r, j), x2 = get_comp(f.a, j), x3 = get_comp(f.q, j);
              if (feasible(c, sp, u0 + j, x0, x1, x3, f.info[j]) && topsis32(tp, x0, x1, x2, x3) >= thr) {
                double rr = topsis64(tp, x0, x1, x2, x3);
                if (rr > bv || (rr == bv && u0 + j < bj)) { bv = rr; bj = u0 + j; }
              }
            }
          }
          warp_argmax64(bv, bj);
          best = bj;
          ws.fp64 += 1;
        }
        // ---- a8: commit (lane 0 writes the overlay; paths searched warp-wide)
        const int nos0 = w->nos, nol0 = w->nol;
        c.ulog_n = 0;
        int fail = 0;
        if (lane == 0) {
          int s = os_slot(c, best);
          int cu = s >= 0 ? w->os_cpu[s] : c.cpu[best];
          int ru = s >= 0 ? w->os_ram[s] : c.ram[best];
          int qu = s >= 0 ? w->os_acc[s] : c.acc[best];
          if (!set_server(c, best, cu - dc, ru - dr, 1, qu)) fail = 2;
        }
        fail = __shfl_sync(NACS_FULL, fail, 0);
        __syncwarp();
        for (int fi = 0; fi < nflow && !fail; ++fi) {
          const int v = w->fv[fi], D = w->fD[fi];
          if (v == best) {
            if (lane == 0) w->fpath[fi] = -1;
            __syncwarp();
            continue;
          }
          int2 wp = wpath(c, best, v);
          if (lane == 0) {
            int su = os_slot(c, best), sv = os_slot(c, v);
            int au = w->os_acc[su];  // best is overlaid above
            int av = sv >= 0 ? w->os_acc[sv] : c.acc[v];
            int bott = min(min(au, av), wp.y);
            if (bott < D) {
              fail = 1;
            } else {
              bool ok = set_server(c, best, w->os_cpu[su], w->os_ram[su], w->os_act[su], au - D);
              int sv2 = os_slot(c, v);
              int cv = sv2 >= 0 ? w->os_cpu[sv2] : c.cpu[v], rv = sv2 >= 0 ? w->os_ram[sv2] : c.ram[v];
              int tv = sv2 >= 0 ? w->os_act[sv2] : c.act[v];
              ok = ok && set_server(c, v, cv, rv, tv, av - D);
              int fid[4];
              int m = path_fids(c, best, v, wp.x, fid);
              for (int t = 0; t < m && ok; ++t) ok = set_link(c, fid[t], fab_val(c, fid[t]) - D);
              if (!ok) fail = 2;
              w->fpath[fi] = wp.x;
            }
          }
          fail = __shfl_sync(NACS_FULL, fail, 0);
          __syncwarp();
        }
        if (fail == 2) { defer = true; break; }  // overlay overflow: the CTA kernel takes it
        if (fail == 1) {  // R18: undo this pod's commit, exclude the server, redo the pod step
          if (lane == 0) {
            undo_commit(c, nos0, nol0);
            if (w->nex < WX) w->ex[w->nex] = best;
            w->nex += 1;
          }
          __syncwarp();
          ws.retries += 1;
          if (w->nex > WX || w->nos + w->nex > WSP) { defer = true; break; }
          continue;
        }
        if (lane == 0) w->pod_srv[p] = best;
        __syncwarp();
        // vlinks of this pod step record their flow's path
        if (hv0) {
          int other = (pa0 == p && pb0 < p) ? pb0 : ((pb0 == p && pa0 < p) ? pa0 : -1);
          if (other >= 0) {
            int v = w->pod_srv[other];
            for (int i = 0; i < nflow; ++i) if (w->fv[i] == v) path0 = w->fpath[i];
          }
        }
        if (hv1) {
          int other = (pa1 == p && pb1 < p) ? pb1 : ((pb1 == p && pa1 < p) ? pa1 : -1);
          if (other >= 0) {
            int v = w->pod_srv[other];
            for (int i = 0; i < nflow; ++i) if (w->fv[i] == v) path1 = w->fpath[i];
          }
        }
        break;
      }
    }
    if (defer) {
      if (lane == 0) deferred[atomicAdd(n_deferred, 1)] = r;
      for (int i = lane; i < nDW; i += 32) c.dirty[i] = 0u;
      __syncwarp();
      continue;
    }
    if (rejected) {
      if (hc) { O.server[c0 + lane] = -1; O.cpu_a[c0 + lane] = 0; O.ram_a[c0 + lane] = 0; }
      if (hv0) { O.bw_a[v0 + lane] = 0; O.path[v0 + lane] = -1; }
      if (hv1) { O.bw_a[v0 + lane + 32] = 0; O.path[v0 + lane + 32] = -1; }
      if (lane == 0) O.status[r] = 0;
      for (int i = lane; i < nDW; i += 32) c.dirty[i] = 0u;
      __syncwarp();
      continue;
    }
    // ---- a9: top-up (R19), containers in index order then vlinks in index order
    int my_ec = 0, my_er = 0;
    for (int i = 0; i < nC; ++i) {
      int pd = __shfl_sync(NACS_FULL, cpod, i);
      int xc = __shfl_sync(NACS_FULL, cmax - cmin, i), xr = __shfl_sync(NACS_FULL, rmax - rmin, i);
      int ec = 0, er = 0;
      if (lane == 0) {
        int u = w->pod_srv[pd];
        int s = os_slot(c, u);  // a placed server is always overlaid
        ec = min(xc, w->os_cpu[s]);
        er = min(xr, w->os_ram[s]);
        w->os_cpu[s] -= ec;
        w->os_ram[s] -= er;
      }
      ec = __shfl_sync(NACS_FULL, ec, 0);
      er = __shfl_sync(NACS_FULL, er, 0);
      if (lane == i) { my_ec = ec; my_er = er; }
    }
    __syncwarp();
    int my_bw0 = 0, my_bw1 = 0;
    for (int e = 0; e < nV; ++e) {
      const int src_lane = e & 31;
      const bool hi = e >= 32;
      int es = __shfl_sync(NACS_FULL, hi ? pa1 : pa0, src_lane);
      int ed = __shfl_sync(NACS_FULL, hi ? pb1 : pb0, src_lane);
      int bmin = __shfl_sync(NACS_FULL, hi ? bn1 : bn0, src_lane);
      int bmax = __shfl_sync(NACS_FULL, hi ? bx1 : bx0, src_lane);
      int pid = __shfl_sync(NACS_FULL, hi ? path1 : path0, src_lane);
      int bw = 0;
      if (lane == 0) {
        int us = w->pod_srv[es], ud = w->pod_srv[ed];
        if (us == ud) {
          bw = bmax;
        } else {
          int ss = os_slot(c, us), sd = os_slot(c, ud);
          int fid[4];
          int m = path_fids(c, us, ud, pid, fid);
          int resid = min(w->os_acc[ss], w->os_acc[sd]);
          for (int t = 0; t < m; ++t) resid = min(resid, fab_val(c, fid[t]));
          int extra = min(bmax - bmin, resid);
          if (extra) {
            w->os_acc[ss] -= extra;
            w->os_acc[sd] -= extra;
            for (int t = 0; t < m; ++t) set_link(c, fid[t], fab_val(c, fid[t]) - extra, false);  // overlaid already
          }
          bw = bmin + extra;
        }
      }
      bw = __shfl_sync(NACS_FULL, bw, 0);
      if (lane == src_lane) { if (hi) my_bw1 = bw; else my_bw0 = bw; }
    }
    // emit M_c, M_ec, c^a, bw^a
    if (hc) {
      O.server[c0 + lane] = w->pod_srv[cpod];
      O.cpu_a[c0 + lane] = cmin + my_ec;
      O.ram_a[c0 + lane] = rmin + my_er;
    }
    if (hv0) {
      bool intra = w->pod_srv[pa0] == w->pod_srv[pb0];
      O.bw_a[v0 + lane] = my_bw0;
      O.path[v0 + lane] = intra ? -1 : path0;
    }
    if (hv1) {
      bool intra = w->pod_srv[pa1] == w->pod_srv[pb1];
      O.bw_a[v0 + lane + 32] = my_bw1;
      O.path[v0 + lane + 32] = intra ? -1 : path1;
    }
    if (lane == 0) O.status[r] = 1;
    for (int i = lane; i < nDW; i += 32) c.dirty[i] = 0u;
    __syncwarp();
  }
  if (lane == 0) {
    if (ws.steps) atomicAdd(&stats[ST_POD_STEPS], ws.steps);
    if (ws.retries) atomicAdd(&stats[ST_RETRIES], ws.retries);
    if (ws.fp64) atomicAdd(&stats[ST_FP64], ws.fp64);
    if (ws.invalid) atomicAdd(&stats[ST_INVALID], ws.invalid);
    if (ws.feas) atomicAdd(&stats[ST_FEAS], ws.feas);
  }
}

// ------------------------------------------------------------------- host ----
static size_t warp_snapshot_bytes(const Geo& g, bool u16) {
  size_t npad = (size_t)((g.n + 127) & ~127);
  size_t nfab = (size_t)g.E * g.h + (size_t)g.k * g.h * g.h;
  return 16 * npad + (((u16 ? 2 : 4) * nfab + 15) & ~(size_t)15);
}
static size_t warp_scratch_bytes(const Geo& g) {
  int nDW = (g.E + g.k * g.h + 31) >> 5, nEW = (g.E + 31) >> 5;
  return ((sizeof(WScr) + 4 * (size_t)(nDW + nEW + g.k)) + 15) & ~(size_t)15;
}

int warp_kernel_warps(const Geo& g) {
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  bool u16 = g.link_cap <= 65535;
  size_t snap = warp_snapshot_bytes(g, u16), per = warp_scratch_bytes(g);
  if (snap + 4 * per + 64 > (size_t)optin) return 0;
  int W = (int)(((size_t)optin - snap - 64) / per);
  return W > 16 ? 16 : W;
}

size_t warp_ulog_entries(int grid, int warps) { return (size_t)grid * warps * WLOG; }

cudaError_t launch_batch_warp(const Geo& g, const Opt& o, const int* d_state, const ReqsDev& R, const OutDev& O,
                              int4* ulog, int* next, int* deferred, int* n_deferred, unsigned long long* stats,
                              int grid, int warps, cudaStream_t st) {
  bool u16 = g.link_cap <= 65535;
  size_t smem = warp_snapshot_bytes(g, u16) + (size_t)warps * warp_scratch_bytes(g);
  if (u16) {
    cudaFuncSetAttribute(k_batch_warp<uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_batch_warp<uint16_t><<<grid, warps * 32, smem, st>>>(g, o, d_state, R, O, ulog, next, deferred, n_deferred,
                                                           stats);
  } else {
    cudaFuncSetAttribute(k_batch_warp<int>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_batch_warp<int><<<grid, warps * 32, smem, st>>>(g, o, d_state, R, O, ulog, next, deferred, n_deferred, stats);
  }
  return cudaGetLastError();
}

}  // namespace nacs
