// nacs_warp.cu — warp-per-request TOPSIS batch kernel (nacs_schedule_batch fast path).
//
// Every warp schedules whole requests on its own: all warps of a CTA share one read-only
// copy of the snapshot in shared memory (criteria in 128-slot tiles of a chunk layout with
// a summary per tile, fabric links as u16), and each warp keeps a private *overlay* of the
// servers and links its current request has modified (R21 snapshot isolation).  Pass A
// (filter + statistics) takes wholly feasible tiles from their summaries and scans the
// others, 128 slots per warp iteration (4 slots per lane, int4 loads); pass B (closeness +
// argmax) visits tiles best-first by a lower bound of q and stops when no unvisited tile
// can hold the best.  The few servers that are special in a pod step (overlaid, excluded
// or flow endpoints) are masked out of the tiles and handled in a parallel specials pass.
// Fabric-table rows touched by the overlay are flagged dirty and read through it.  The
// warps advance in lockstep groups of 8 (named barriers) so that a group runs one code
// region at a time.
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
constexpr int WDW = 40;   // dirty-row bitmap words: fabric rows E + k*h = k^2 <= 1280 (k <= 35)
constexpr int WEW = 20;   // edge bitmap words: E = k^2/2 <= 640
constexpr int WCH = 96;   // chunks of 128 slots: n <= 12288
constexpr int WWARPS = 16; // warps per CTA (static per-warp scratch)
#ifndef NACS_WARP_THREADS  // threads of k_batch_warp (<= 32 WWARPS); the register budget is 64K / this
#define NACS_WARP_THREADS 512
#endif
static_assert(NACS_WARP_THREADS % 32 == 0 && NACS_WARP_THREADS <= 32 * WWARPS, "k_batch_warp threads");
}  // namespace

struct __align__(16) WScr {
  int nos, nol, nflow, sumD, G, nsp, nex, pad0;
  int os_u[WOS], os_cpu[WOS], os_ram[WOS], os_act[WOS], os_acc[WOS];
  int ol_id[WOL], ol_val[WOL];
  int pod_srv[WC];
  int fv[WF], fD[WF], fok[WF], fpath[WF];
  union {
    struct {
      int sp_u[WSP], sp_info[WSP];
    };
    int dem[WOL + WOS];  // finish_request: top-up demands (the special list is free by then)
  };
  int ex[WX];
  int os_pos[WOS], ex_pos[WX];  // their slots in the chunk layout
  unsigned slow[4];  // chunks of 128 slots the scans take on the slow path (<= 128 chunks)
  unsigned none_m[4];  // chunks without a feasible server in this pod step (pass A)
  unsigned sp_has[4];  // chunks holding a special server
  unsigned eb_has[4];  // chunks holding a server under a fabric-blocked edge switch
  unsigned char sp_first[WCH];  // index in sp_u of a chunk's first special (valid where sp_has)
  int net;
  TopsisP tp0;            // R25: the first pod step's TOPSIS parameters
  int dc0, dr0;           // and its CPU / RAM demand (its feasible set, no flows yet)
  unsigned dirty[WDW];    // fabric rows (edge-agg rows, then agg-core rows) the overlay touched
  unsigned edgebad[WEW];  // edge switches without a feasible fabric path this pod step
};

// Static summary of one 128-slot chunk of the layout (k_warp_layout): the box of its
// criteria (CPU, RAM, access link; f_u as bits: 1 = has 0, 2 = has 1) and the exact
// aggregates pass A needs when the whole chunk is feasible.
struct ChunkT {
  int lo[3];
  int act;
  int hi[3];
  int cnt;
  int nact, pad;
  unsigned long long sq[3];
};
static_assert(sizeof(ChunkT) == 64, "ChunkT is 16 words");

template <typename LT>
struct WCtx {
  int k, h, n, npad, E, nfabea;  // nfabea = E*h (start of agg-core links in fab[])
  unsigned magic;
  const int* snap;  // criteria in 128-slot tiles: cpu[128] | ram[128] | (server << 1 | f_u)[128] | acc[128] (shared)
  const ChunkT* ctab;  // [nch] chunk summaries (shared)
  const int* inv;      // server -> slot (global)
  int nch;
  const LT* fab;                           // edge-agg[E*h] | agg-core[k*h*h] (shared)
  WScr* w;
  int4* ulog;
  int ulog_n;
  int lane;
  int nDW;
  int fabmin;  // smallest fabric residual of the snapshot
  unsigned a_snap;  // 32-bit shared address of the criteria tiles + 16 * lane
  Opt o;
};

// criterion j (0 cpu, 1 ram, 2 act, 3 acc) of server u in the tiled shared snapshot
__device__ __forceinline__ int tile_idx(int u, int j) { return ((u >> 7) << 9) + (j << 7) + (u & 127); }

__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
// read-only snapshot loads through explicit shared-window addresses
__device__ __forceinline__ int4 lds128(unsigned a) {
  int4 v;
  asm("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ unsigned lds32v(unsigned a) {
  unsigned v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}

// ------------------------------------------------------------ overlay reads --
// The link overlay is kept sorted by fabric link id: per-lane lookups binary-search it.
__device__ __forceinline__ int ol_find(const WScr* w, int fid) {
  int lo = 0, hi = w->nol;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (w->ol_id[mid] < fid) lo = mid + 1;
    else hi = mid;
  }
  return (lo < w->nol && w->ol_id[lo] == fid) ? lo : -1;
}
template <typename LT>
__device__ __forceinline__ bool row_dirty(const WCtx<LT>& c, int row) {
  return (c.w->dirty[row >> 5] >> (row & 31)) & 1u;
}
// fabric link fid (per lane): the overlay value if its row is dirty and it is overlaid
template <typename LT>
__device__ __forceinline__ int fab_val(const WCtx<LT>& c, int fid) {
  int v = (int)c.fab[fid];
  if (row_dirty(c, (int)div_h((unsigned)fid, c.magic))) {
    int s = ol_find(c.w, fid);
    if (s >= 0) v = c.w->ol_val[s];
  }
  return v;
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
// overlay slot of server u, -1 if none (warp-cooperative, u uniform)
template <typename LT>
__device__ __forceinline__ int w_slot(const WCtx<LT>& c, int u) {
  const WScr* w = c.w;
  unsigned m = __ballot_sync(NACS_FULL, c.lane < w->nos && w->os_u[c.lane] == u);
  return m ? __ffs(m) - 1 : -1;
}
template <typename LT>
__device__ __forceinline__ int acc_val(const WCtx<LT>& c, int u) {
  int s = os_slot(c, u);
  return s >= 0 ? c.w->os_acc[s] : c.snap[tile_idx(c.inv[u], 3)];
}

// -------------------------------------------- overlay writes (warp-cooperative) --
// All lanes call with uniform arguments; lane 0 writes.  Returns false on overflow.
template <typename LT>
__device__ bool w_set_server(WCtx<LT>& c, int u, int pos, int cpu, int ram, int act, int acc, bool log = true) {
  WScr* w = c.w;
  const int s0 = w_slot(c, u);  // uniform
  bool ok = true;
  if (s0 < 0 && w->nos >= WOS) ok = false;
  if (s0 >= 0 && log && c.ulog_n >= WLOG) ok = false;
  __syncwarp();
  if (ok && c.lane == 0) {
    int s = s0;
    if (s < 0) {
      s = w->nos++;
      w->os_u[s] = u;
      w->os_pos[s] = pos;
    } else if (log) {
      c.ulog[c.ulog_n] = make_int4(s, w->os_cpu[s], w->os_ram[s], w->os_acc[s] * 2 + w->os_act[s]);
    }
    w->os_cpu[s] = cpu;
    w->os_ram[s] = ram;
    w->os_act[s] = act;
    w->os_acc[s] = acc;
  }
  if (ok && log && s0 >= 0) c.ulog_n += 1;
  __syncwarp();
  return ok;
}
template <typename LT>
// Link fid (fabric) += delta on the current residual (overlay value, else the snapshot's).
__device__ bool w_add_link(WCtx<LT>& c, int fid, int delta, bool log = true) {
  WScr* w = c.w;
  const int nol = w->nol;
  int pos = 0;
  bool found = false;
#pragma unroll
  for (int q = 0; q < WOL / 32; ++q) {
    const int j = c.lane + 32 * q;
    const int id = j < nol ? w->ol_id[j] : INT_MAX;
    pos += __popc(__ballot_sync(NACS_FULL, id < fid));
    found |= __any_sync(NACS_FULL, id == fid);
  }
  if (!found && nol >= WOL) return false;
  if (log && c.ulog_n >= WLOG) return false;
  if (found) {
    if (c.lane == 0) {
      if (log) c.ulog[c.ulog_n] = make_int4(-1, fid, w->ol_val[pos], 0);
      w->ol_val[pos] += delta;
    }
  } else {  // insert at pos, shifting the tail right
    const int val = (int)c.fab[fid] + delta;
    int ids[WOL / 32], vals[WOL / 32];
#pragma unroll
    for (int q = 0; q < WOL / 32; ++q) {
      const int j = c.lane + 32 * q;
      ids[q] = j < nol ? w->ol_id[j] : 0;
      vals[q] = j < nol ? w->ol_val[j] : 0;
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < WOL / 32; ++q) {
      const int j = c.lane + 32 * q;
      if (j < nol && j >= pos) { w->ol_id[j + 1] = ids[q]; w->ol_val[j + 1] = vals[q]; }
    }
    __syncwarp();
    if (c.lane == 0) {
      w->ol_id[pos] = fid;
      w->ol_val[pos] = val;
      w->nol = nol + 1;
      if (log) c.ulog[c.ulog_n] = make_int4(-1, fid, 0, 1);
    }
  }
  if (log) c.ulog_n += 1;
  if (c.lane == 0) {
    unsigned row = div_h((unsigned)fid, c.magic);
    c.w->dirty[row >> 5] |= 1u << (row & 31);
  }
  __syncwarp();
  return true;
}
// Undo this pod step's commit (R18): restore in reverse order.  Warp-cooperative.
template <typename LT>
__device__ void w_undo(WCtx<LT>& c, int nos0) {
  WScr* w = c.w;
  for (int i = c.ulog_n - 1; i >= 0; --i) {
    int4 e = make_int4(0, 0, 0, 0);
    if (c.lane == 0) e = c.ulog[i];
    e.x = __shfl_sync(NACS_FULL, e.x, 0);
    e.y = __shfl_sync(NACS_FULL, e.y, 0);
    e.z = __shfl_sync(NACS_FULL, e.z, 0);
    e.w = __shfl_sync(NACS_FULL, e.w, 0);
    if (e.x >= 0) {
      if (c.lane == 0) {
        w->os_cpu[e.x] = e.y;
        w->os_ram[e.x] = e.z;
        w->os_acc[e.x] = e.w >> 1;
        w->os_act[e.x] = e.w & 1;
      }
    } else {
      const int pos = ol_find(w, e.y);
      if (!e.w) {
        if (c.lane == 0) w->ol_val[pos] = e.z;
      } else {  // the link was inserted by this commit: remove it
        const int nol = w->nol;
        int ids[WOL / 32], vals[WOL / 32];
#pragma unroll
        for (int q = 0; q < WOL / 32; ++q) {
          const int j = c.lane + 32 * q;
          ids[q] = j < nol ? w->ol_id[j] : 0;
          vals[q] = j < nol ? w->ol_val[j] : 0;
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < WOL / 32; ++q) {
          const int j = c.lane + 32 * q;
          if (j < nol && j > pos) { w->ol_id[j - 1] = ids[q]; w->ol_val[j - 1] = vals[q]; }
        }
        if (c.lane == 0) w->nol = nol - 1;
      }
    }
    __syncwarp();
  }
  if (c.lane == 0) w->nos = nos0;
  c.ulog_n = 0;
  __syncwarp();
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
// Lane a < h holds min(EA[eu][a], EA[ev][a]) (h <= 32); cross-pod paths (a, b) read it by
// shuffle, so each edge-aggregation residual is looked up once.
template <typename LT>
__device__ int2 wpath(const WCtx<LT>& c, int u, int v) {
  const int h = c.h;
  const int eu = (int)div_h(u, c.magic), ev = (int)div_h(v, c.magic);
  if (eu == ev) return make_int2(0, INT_MAX);
  const int pu = (int)div_h(eu, c.magic), pv = (int)div_h(ev, c.magic);
  const int eav = c.lane < h ? min(fab_val(c, eu * h + c.lane), fab_val(c, ev * h + c.lane)) : -1;
  int best = -1, bt = INT_MAX;
  if (pu == pv) {
    if (c.lane < h) { best = eav; bt = c.lane; }
  } else {
    const int hh = h * h;
    for (int t0 = 0; t0 < hh; t0 += 32) {
      const int t = t0 + c.lane;
      const int a = t < hh ? (int)div_h(t, c.magic) : 0, b = t - a * h;
      const int ea = __shfl_sync(NACS_FULL, eav, a);
      if (t < hh) {
        const int x = min(ea, min(fab_val(c, c.nfabea + (pu * h + a) * h + b), fab_val(c, c.nfabea + (pv * h + a) * h + b)));
        if (x > best) { best = x; bt = t; }
      }
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

// Is some core switch (a, b) joined to pods p and pv by links both >= D?  (per lane)
template <typename LT>
__device__ __forceinline__ bool core_ok(const WCtx<LT>& c, int p, int pv, int a, int D) {
  const int h = c.h;
  const int f1 = c.nfabea + (p * c.h + a) * h, f2 = c.nfabea + (pv * c.h + a) * h;
  if (!row_dirty(c, c.E + p * h + a) && !row_dirty(c, c.E + pv * h + a)) {
    const LT* r1 = c.fab + f1;
    const LT* r2 = c.fab + f2;
    for (int b = 0; b < h; ++b)
      if ((int)r1[b] >= D && (int)r2[b] >= D) return true;
    return false;
  }
  for (int b = 0; b < h; ++b)
    if (fab_val(c, f1 + b) >= D && fab_val(c, f2 + b) >= D) return true;
  return false;
}

// a2: mark the edge switches from which some flow's widest fabric bottleneck is below its
// demand: edge e reaches edge(v) iff some aggregation index a has EA[e][a] >= D,
// EA[ev][a] >= D and (other pod) some core (a, b) with both agg-core links >= D.
// Each lane tests its edges with early exit on the first feasible (a, b).
template <typename LT>
__device__ void wfabric(WCtx<LT>& c) {
  WScr* w = c.w;
  const int h = c.h, E = c.E;
  const int nEW = (E + 31) >> 5;
  for (int i = c.lane; i < nEW; i += 32) c.w->edgebad[i] = 0u;
  // every fabric link (snapshot and overlay) >= D: no edge is cut off for that flow
  int lmin = c.fabmin;
  for (int i = c.lane; i < w->nol; i += 32) lmin = min(lmin, w->ol_val[i]);
  lmin = __reduce_min_sync(NACS_FULL, lmin);
  __syncwarp();
  for (int f = 0; f < w->nflow; ++f) {
    const int v = w->fv[f], D = w->fD[f];
    if (D <= lmin) continue;
    const int ev = (int)div_h(v, c.magic), pv = (int)div_h(ev, c.magic);
    // vm: aggregation switches a with EA[ev][a] >= D
    const bool vme = c.lane < h && fab_val(c, ev * h + c.lane) >= D;
    const unsigned vm = __ballot_sync(NACS_FULL, vme);
    for (int e0 = 0; e0 < E; e0 += 32) {
      const int e = e0 + c.lane;
      bool bad = false;
      if (e < E && e != ev) {
        const int pe = (int)div_h(e, c.magic);
        const bool dirty = row_dirty(c, e);
        bool ok = false;
        for (unsigned m = vm; m && !ok; m &= m - 1) {
          const int a = __ffs(m) - 1;
          const int ea = dirty ? fab_val(c, e * h + a) : (int)c.fab[e * h + a];
          if (ea < D) continue;
          ok = pe == pv || core_ok(c, pe, pv, a, D);
        }
        bad = !ok;
      }
      const unsigned bw = __ballot_sync(NACS_FULL, bad);
      if (c.lane == 0) c.w->edgebad[e0 >> 5] |= bw;
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------------ scans ----
// Filter parameters of one pod step (a3).  For ordinary servers the network conditions
// fold into thresholds: sumDp = sumD (INT_MIN without path filter) and dcp = dc
// (INT_MAX when some flow's own access link is short, G false).
struct StepP {
  int dc, dr, dcp, sumDp;
  bool net, pf, h4;
  // R25 walk (pod steps after the first): ordinary servers must also be in the first pod
  // step's feasible set (snapshot CPU >= f0c, RAM >= f0r) -- folded into tc, tr
  bool walk;
  int f0c, f0r;
  int tc, tr;  // CPU / RAM thresholds of ordinary servers: max(dcp, f0c), max(dr, f0r)
};

template <typename LT>
__device__ __forceinline__ unsigned ebad(const WCtx<LT>& c, unsigned u) {
  unsigned e = div_h(u, c.magic);
  return (c.w->edgebad[e >> 5] >> (e & 31)) & 1u;
}
// edge-infeasibility bits (bit j) of the lane's servers u0..u0+3
template <typename LT>
__device__ __forceinline__ unsigned ebad4(const WCtx<LT>& c, const StepP& sp, unsigned u0) {
  if (!sp.net) return 0u;
  if (sp.h4) return ebad(c, u0) ? 0xFu : 0u;
  return ebad(c, u0) | (ebad(c, u0 + 1) << 1) | (ebad(c, u0 + 2) << 2) | (ebad(c, u0 + 3) << 3);
}
__device__ __forceinline__ bool ok_plain(const StepP& sp, int x0, int x1, int x3, unsigned bad) {
  return (x0 >= sp.tc) & (x1 >= sp.tr) & (x3 >= sp.sumDp) & (bad == 0u);
}
// a special server: excluded (R18), a flow endpoint (its own flow uses the host bus), or
// only overlaid (ordinary rule on its overlay values)
template <typename LT>
__device__ __forceinline__ bool ok_special(const WCtx<LT>& c, const StepP& sp, int x0, int x1, int x3,
                                           unsigned bad, int info) {
  if (info & 64) return false;
  int f = (info >> 7) - 1;
  if (f >= 0) return (x0 >= sp.dc) & (x1 >= sp.dr) & (!sp.pf || c.w->fok[f]);
  return ok_plain(sp, x0, x1, x3, bad);
}

struct AccA {
  int nf, nact;
  unsigned mn0, mn1, mn3, mx0, mx1, mx3;
  unsigned long long q0, q1, q3;
};
// a4: statistics over F, branch-free
__device__ __forceinline__ void acc_a(AccA& a, bool ok, int x0, int x1, int x2, int x3) {
  unsigned o0 = ok ? (unsigned)x0 : 0u, o1 = ok ? (unsigned)x1 : 0u, o3 = ok ? (unsigned)x3 : 0u;
  a.nf += ok ? 1 : 0;
  a.nact += ok ? (x2 & 1) : 0;
  a.mx0 = max(a.mx0, o0);
  a.mx1 = max(a.mx1, o1);
  a.mx3 = max(a.mx3, o3);
  a.mn0 = min(a.mn0, ok ? o0 : UINT_MAX);
  a.mn1 = min(a.mn1, ok ? o1 : UINT_MAX);
  a.mn3 = min(a.mn3, ok ? o3 : UINT_MAX);
  a.q0 += (unsigned long long)o0 * o0;
  a.q1 += (unsigned long long)o1 * o1;
  a.q3 += (unsigned long long)o3 * o3;
}
// a7: per-lane best (smallest q = largest closeness, lowest server index) and second best;
// chunks are visited in any order, so equal q compare server indices
struct AccB {
  float b1, b2;
  int i1, p1;  // server index and slot of b1
};
__device__ __forceinline__ void acc_b(AccB& b, bool ok, float q, int id, int pos) {
  const float qe = ok ? q : __int_as_float(0x7f800000);
  const bool lt = qe < b.b1 || (qe == b.b1 && qe != __int_as_float(0x7f800000) && (unsigned)id < (unsigned)b.i1);
  b.b2 = lt ? b.b1 : fminf(b.b2, qe);
  b.i1 = lt ? id : b.i1;
  b.p1 = lt ? pos : b.p1;
  b.b1 = lt ? qe : b.b1;
}
// merge accumulator o (a disjoint set of servers) into a: lowest index on equal q
__device__ __forceinline__ void merge_b(AccB& a, const AccB& o) {
  const bool lt = o.b1 < a.b1 || (o.b1 == a.b1 && (unsigned)o.i1 < (unsigned)a.i1);
  a.b2 = fminf(fminf(a.b2, o.b2), lt ? a.b1 : o.b1);
  a.i1 = lt ? o.i1 : a.i1;
  a.p1 = lt ? o.p1 : a.p1;
  a.b1 = lt ? o.b1 : a.b1;
}


__device__ __forceinline__ bool slow_bit(const unsigned* m, int ch) { return (m[ch >> 5] >> (ch & 31)) & 1u; }

// Masks of the lane's 4 slots of chunk ch (bit j = slot 4 lane + j): `skip` = special
// servers (taken by the specials pass instead), `bad` = servers under an edge switch
// without a feasible fabric path.  Both 0 for clean chunks.
template <typename LT>
__device__ __forceinline__ void chunk_masks(const WCtx<LT>& c, const StepP& sp, int ch, const int4& A,
                                            unsigned& skip, unsigned& bad) {
  const WScr* w = c.w;
  skip = 0u;
  bad = 0u;
  if (!slow_bit(w->slow, ch)) return;
  const int base = ch << 7;
  if (slow_bit(w->sp_has, ch)) {
    for (int t = w->sp_first[ch]; t < w->nsp && w->sp_u[t] < base + 128; ++t) {
      const int d = w->sp_u[t] - base;
      if ((d >> 2) == c.lane) skip |= 1u << (d & 3);
    }
  }
  if (sp.net && slow_bit(w->eb_has, ch)) {
    bad = ebad(c, (unsigned)A.x >> 1) | (ebad(c, (unsigned)A.y >> 1) << 1) | (ebad(c, (unsigned)A.z >> 1) << 2) |
          (ebad(c, (unsigned)A.w >> 1) << 3);
  }
}

// Special server t of the step (lanes in parallel): current values (overlay, else the
// snapshot at its slot), server index, feasibility by the special rules.
template <typename LT>
__device__ __forceinline__ bool special_vals(const WCtx<LT>& c, const StepP& sp, int t, int& x0, int& x1, int& x2,
                                            int& x3, int& id) {
  const WScr* w = c.w;
  const int pos = w->sp_u[t], inf = w->sp_info[t];
  const int slot = (inf & 63) - 1;
  if (slot >= 0) {
    x0 = w->os_cpu[slot];
    x1 = w->os_ram[slot];
    id = w->os_u[slot];
    x2 = (id << 1) | w->os_act[slot];
    x3 = w->os_acc[slot];
  } else {
    x0 = c.snap[tile_idx(pos, 0)];
    x1 = c.snap[tile_idx(pos, 1)];
    x2 = c.snap[tile_idx(pos, 2)];
    x3 = c.snap[tile_idx(pos, 3)];
    id = x2 >> 1;
  }
  const unsigned bad = sp.net ? ebad(c, (unsigned)id) : 0u;
  return ok_special(c, sp, x0, x1, x3, bad, inf);
}

// R25 walk: a special server is scored on its snapshot values (the request-start state
// the first pod step ranked) and must have been in that step's feasible set.
template <typename LT>
__device__ __forceinline__ void walk_vals(const WCtx<LT>& c, const StepP& sp, int pos, bool& ok, int& x0, int& x1,
                                          int& x2, int& x3) {
  x0 = c.snap[tile_idx(pos, 0)];
  x1 = c.snap[tile_idx(pos, 1)];
  x2 = c.snap[tile_idx(pos, 2)];
  x3 = c.snap[tile_idx(pos, 3)];
  ok = ok && x0 >= sp.f0c && x1 >= sp.f0r;
}

// Pass A (a3 + a4): filter and statistics.  Per chunk (one lane each): a chunk whose box
// lies inside the thresholds and holds no special server is feasible as a whole and adds
// its precomputed aggregates; a chunk whose box misses a threshold holds no feasible
// server; the warp scans the others, 128 slots per iteration, and the special servers
// in one parallel pass.  Exact either way.
template <typename LT>
__device__ void pass_a(const WCtx<LT>& c, const StepP& sp, AccA& a, unsigned long long& scanned) {
  WScr* w = c.w;
  unsigned scan_m[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int ch = c.lane + 32 * i;
    bool sc = false, none = false;
    if (ch < c.nch) {
      const bool slow = (w->slow[i] >> c.lane) & 1u;
      const ChunkT& t = c.ctab[ch];
      const bool full = !slow && t.cnt > 0 && t.lo[0] >= sp.tc && t.lo[1] >= sp.tr && t.lo[2] >= sp.sumDp;
      none = !slow && (t.cnt == 0 || t.hi[0] < sp.tc || t.hi[1] < sp.tr || t.hi[2] < sp.sumDp);
      sc = !full && !none;
      if (full) {
        a.nf += t.cnt;
        a.nact += t.nact;
        a.mx0 = max(a.mx0, (unsigned)t.hi[0]); a.mn0 = min(a.mn0, (unsigned)t.lo[0]);
        a.mx1 = max(a.mx1, (unsigned)t.hi[1]); a.mn1 = min(a.mn1, (unsigned)t.lo[1]);
        a.mx3 = max(a.mx3, (unsigned)t.hi[2]); a.mn3 = min(a.mn3, (unsigned)t.lo[2]);
        a.q0 += t.sq[0];
        a.q1 += t.sq[1];
        a.q3 += t.sq[2];
      }
    }
    scan_m[i] = __ballot_sync(NACS_FULL, sc);
    const unsigned nm = __ballot_sync(NACS_FULL, none);
    if (c.lane == 0) w->none_m[i] = nm;
  }
#pragma unroll 1
  for (int i = 0; i < 4; ++i) {
    for (unsigned m = scan_m[i]; m; m &= m - 1) {
      const int ch = 32 * i + __ffs(m) - 1;
      scanned += 128;
      const unsigned ao = c.a_snap + ((unsigned)ch << 11);
      const int4 C = lds128(ao), Rm = lds128(ao + 512), A = lds128(ao + 1024), Q = lds128(ao + 1536);
      unsigned skip, bad;
      chunk_masks(c, sp, ch, A, skip, bad);
      const unsigned off = skip | bad;
      acc_a(a, ok_plain(sp, C.x, Rm.x, Q.x, off & 1u), C.x, Rm.x, A.x, Q.x);
      acc_a(a, ok_plain(sp, C.y, Rm.y, Q.y, off & 2u), C.y, Rm.y, A.y, Q.y);
      acc_a(a, ok_plain(sp, C.z, Rm.z, Q.z, off & 4u), C.z, Rm.z, A.z, Q.z);
      acc_a(a, ok_plain(sp, C.w, Rm.w, Q.w, off & 8u), C.w, Rm.w, A.w, Q.w);
    }
  }
  for (int t = c.lane; t < w->nsp; t += 32) {
    int x0, x1, x2, x3, id;
    const bool ok = special_vals(c, sp, t, x0, x1, x2, x3, id);
    acc_a(a, ok, x0, x1, x2, x3);
  }
  __syncwarp();
}

// R25 walk, pass A: no statistics (the first pod step's order is fixed); only the chunks
// that cannot hold an admitted server of that order.
template <typename LT>
__device__ void pass_a_walk(const WCtx<LT>& c, const StepP& sp) {
  WScr* w = c.w;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int ch = c.lane + 32 * i;
    bool none = false;
    if (ch < c.nch) {
      const bool slow = (w->slow[i] >> c.lane) & 1u;
      const ChunkT& t = c.ctab[ch];
      none = !slow && (t.cnt == 0 || t.hi[0] < sp.tc || t.hi[1] < sp.tr || t.hi[2] < sp.sumDp);
    }
    const unsigned nm = __ballot_sync(NACS_FULL, none);
    if (c.lane == 0) w->none_m[i] = nm;
  }
  __syncwarp();
}

// Lower bound of q = Ed+^2 / Ed-^2 over the servers of a chunk (its box clipped to the
// [min, max] of F): Ed+_c >= s_c (max_c - min(hi_c, max_c)), Ed-_c <= s_c (min(hi_c, max_c)
// - min_c).  FP32 with relative error <= 12u; callers prune with a 2^-12 margin.
__device__ __forceinline__ float chunk_qlb(const TopsisP& t, const ChunkT& ct, int act_or = 0) {
  float ep2, em2;
  {
    const int ci[3] = {0, 1, 3};
    float e[3], m[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const int hc = min(ct.hi[c], t.mx[ci[c]]);
      e[c] = t.sf[ci[c]] * (float)(t.mx[ci[c]] - hc);
      m[c] = t.sf[ci[c]] * (float)max(0, hc - t.mn[ci[c]]);
    }
    const int am = ct.act | act_or;
    const float pa = (am & 2) ? ((am & 1) ? fminf(t.p2sq[0], t.p2sq[1]) : t.p2sq[1]) : t.p2sq[0];
    const float ma = (am & 2) ? ((am & 1) ? fmaxf(t.m2sq[0], t.m2sq[1]) : t.m2sq[1]) : t.m2sq[0];
    ep2 = fmaf(e[2], e[2], fmaf(e[1], e[1], fmaf(e[0], e[0], pa)));
    em2 = fmaf(m[2], m[2], fmaf(m[1], m[1], fmaf(m[0], m[0], ma)));
  }
  return em2 > 0.f ? ep2 * rcp_approx(em2) : __int_as_float(0x7f800000);
}
constexpr float kPruneMargin = 1.0f + 2.44140625e-4f;  // 1 + 2^-12

// Scores of the lane's 4 slots of chunk ch into b (a5T + a7); special slots are skipped
// (the specials pass scores them).
template <typename LT>
__device__ __forceinline__ void score_chunk(const WCtx<LT>& c, const StepP& sp, const TopsisP& tp, int ch,
                                            AccB& b) {
  const int p0 = (ch << 7) + 4 * c.lane;
  const unsigned ao = c.a_snap + ((unsigned)ch << 11);
  const int4 C = lds128(ao), Rm = lds128(ao + 512), A = lds128(ao + 1024), Q = lds128(ao + 1536);
  unsigned skip, bad;
  chunk_masks(c, sp, ch, A, skip, bad);
  const unsigned off = skip | bad;
  AccB b2 = {__int_as_float(0x7f800000), __int_as_float(0x7f800000), -1, -1};  // shorter chains
  acc_b(b, ok_plain(sp, C.x, Rm.x, Q.x, off & 1u), topsis_q32_scan(tp, C.x, Rm.x, A.x, Q.x), A.x >> 1, p0);
  acc_b(b2, ok_plain(sp, C.y, Rm.y, Q.y, off & 2u), topsis_q32_scan(tp, C.y, Rm.y, A.y, Q.y), A.y >> 1, p0 + 1);
  acc_b(b, ok_plain(sp, C.z, Rm.z, Q.z, off & 4u), topsis_q32_scan(tp, C.z, Rm.z, A.z, Q.z), A.z >> 1, p0 + 2);
  acc_b(b2, ok_plain(sp, C.w, Rm.w, Q.w, off & 8u), topsis_q32_scan(tp, C.w, Rm.w, A.w, Q.w), A.w >> 1, p0 + 3);
  merge_b(b, b2);
}

// Pass B (a5T + a7): the special servers first (lanes in parallel), then best-first over
// chunks.  Every chunk with a feasible server gets the lower bound of its q from its box
// (its special slots are skipped, so the box holds what the chunk scores); the warp
// visits chunks in increasing bound while the bound is within the prune margin of the
// best q so far.  Every server with q32 <= q1 (1 + 2^-12) is visited, so q1, its server
// and the second best q2 (where q2 - q1 <= delta q1 matters) are those of a full scan.
template <typename LT>
__device__ void pass_b(const WCtx<LT>& c, const StepP& sp, const TopsisP& tp, AccB& b,
                       unsigned long long& scanned) {
  const WScr* w = c.w;
  const float INF = __int_as_float(0x7f800000);
  for (int t = c.lane; t < w->nsp; t += 32) {
    int x0, x1, x2, x3, id;
    bool ok = special_vals(c, sp, t, x0, x1, x2, x3, id);
    if (sp.walk) walk_vals(c, sp, w->sp_u[t], ok, x0, x1, x2, x3);
    acc_b(b, ok, topsis_q32_scan(tp, x0, x1, x2, x3), id, w->sp_u[t]);
  }
  float lb[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int ch = c.lane + 32 * i;
    lb[i] = INF;
    if (ch < c.nch && !((w->none_m[i] >> c.lane) & 1u)) lb[i] = chunk_qlb(tp, c.ctab[ch]);
  }
  float best = __uint_as_float(__reduce_min_sync(NACS_FULL, __float_as_uint(b.b1)));
  for (;;) {
    float m = lb[0];
    int mi = 0;
#pragma unroll
    for (int i = 1; i < 4; ++i)
      if (lb[i] < m) { m = lb[i]; mi = i; }
    // warp argmin of the bounds (non-negative floats order like their bit patterns)
    const unsigned key = __float_as_uint(m);
    const unsigned km = __reduce_min_sync(NACS_FULL, key);
    const float mf = __uint_as_float(km);
    if (!(mf <= best * kPruneMargin) || mf == INF) break;
    const int ch = (int)__reduce_min_sync(NACS_FULL, key == km ? (unsigned)(c.lane + 32 * mi) : 0xffffffffu);
    if (ch == c.lane + 32 * mi) lb[mi] = INF;
    scanned += 128;
    score_chunk(c, sp, tp, ch, b);
    best = __uint_as_float(__reduce_min_sync(NACS_FULL, __float_as_uint(b.b1)));
  }
}

// FP64 re-decision (R14): exact closeness of every feasible server with q32 <= thr (chunks
// whose bound exceeds thr are skipped by the same margin; specials in parallel).
__device__ __forceinline__ void fp64_take(const TopsisP& tp, float thr, bool ok, int x0, int x1, int x2, int x3,
                                          int u, int pos, double& bv, int& bj, int& bp) {
  if (ok && topsis_q32(tp, x0, x1, x2 & 1, x3) <= thr) {
    const double rr = topsis64(tp, x0, x1, x2 & 1, x3);
    if (rr > bv || (rr == bv && u < bj)) { bv = rr; bj = u; bp = pos; }
  }
}
template <typename LT>
__device__ void scan_fp64(const WCtx<LT>& c, const StepP& sp, const TopsisP& tp, float thr, double& bv, int& bj,
                          int& bp) {
  const WScr* w = c.w;
  for (int t = c.lane; t < w->nsp; t += 32) {
    int x0, x1, x2, x3, id;
    bool ok = special_vals(c, sp, t, x0, x1, x2, x3, id);
    if (sp.walk) walk_vals(c, sp, w->sp_u[t], ok, x0, x1, x2, x3);
    fp64_take(tp, thr, ok, x0, x1, x2, x3, id, w->sp_u[t], bv, bj, bp);
  }
  for (int ch = 0; ch < c.nch; ++ch) {
    if (slow_bit(w->none_m, ch)) continue;
    if (!(chunk_qlb(tp, c.ctab[ch]) <= thr * kPruneMargin)) continue;
    const int p0 = (ch << 7) + 4 * c.lane;
    const unsigned ao = c.a_snap + ((unsigned)ch << 11);
    const int4 C = lds128(ao), Rm = lds128(ao + 512), A = lds128(ao + 1024), Q = lds128(ao + 1536);
    unsigned skip, bad;
    chunk_masks(c, sp, ch, A, skip, bad);
    const unsigned off = skip | bad;
    fp64_take(tp, thr, ok_plain(sp, C.x, Rm.x, Q.x, off & 1u), C.x, Rm.x, A.x, Q.x, A.x >> 1, p0, bv, bj, bp);
    fp64_take(tp, thr, ok_plain(sp, C.y, Rm.y, Q.y, off & 2u), C.y, Rm.y, A.y, Q.y, A.y >> 1, p0 + 1, bv, bj, bp);
    fp64_take(tp, thr, ok_plain(sp, C.z, Rm.z, Q.z, off & 4u), C.z, Rm.z, A.z, Q.z, A.z >> 1, p0 + 2, bv, bj, bp);
    fp64_take(tp, thr, ok_plain(sp, C.w, Rm.w, Q.w, off & 8u), C.w, Rm.w, A.w, Q.w, A.w >> 1, p0 + 3, bv, bj, bp);
  }
}

// Build the special list, sorted by slot: overlay servers, excluded servers, flow servers.
template <typename LT>
__device__ void build_specials(WCtx<LT>& c) {
  WScr* w = c.w;
  const int l = c.lane;
  // entry A: overlay slot l; entry B: excluded server l not in the overlay
  bool va = l < w->nos, vbx = false;
  int ua = va ? w->os_pos[l] : INT_MAX, ia = 0;
  if (va) {
    const int su = w->os_u[l];
    bool ex = false;
    for (int i = 0; i < w->nex; ++i) ex |= w->ex[i] == su;
    int f = -1;
    for (int i = 0; i < w->nflow; ++i)
      if (w->fv[i] == su) f = i;
    ia = (l + 1) | (ex ? 64 : 0) | ((f + 1) << 7);
  }
  int ub = INT_MAX;
  if (l < w->nex) {
    vbx = os_slot(c, w->ex[l]) < 0;
    ub = vbx ? w->ex_pos[l] : INT_MAX;
  }
  int ra = 0, rb = 0;
  const int lim = max(w->nos, w->nex);
  for (int s = 0; s < lim; ++s) {
    int xa = __shfl_sync(NACS_FULL, ua, s);
    int xb = __shfl_sync(NACS_FULL, ub, s);
    ra += (xa < ua) + (xb < ua);
    rb += (xa < ub) + (xb < ub);
  }
  if (va) { w->sp_u[ra] = ua; w->sp_info[ra] = ia; }
  if (vbx) { w->sp_u[rb] = ub; w->sp_info[rb] = 64; }
  int cnt = __popc(__ballot_sync(NACS_FULL, va)) + __popc(__ballot_sync(NACS_FULL, vbx));
  if (l == 0) w->nsp = cnt;
  if (l < 4) w->slow[l] = 0u;
  __syncwarp();
  // slow chunks: those holding a special server or, with the path filter on, a server
  // under an edge switch without a feasible fabric path (all others skip both tests)
  for (int i = l; i < cnt; i += 32) {
    const int u = w->sp_u[i], ch = u >> 7;
    atomicOr(&w->slow[ch >> 5], 1u << (ch & 31));
    if (i == 0 || (w->sp_u[i - 1] >> 7) != ch) w->sp_first[ch] = (unsigned char)i;
  }
  __syncwarp();
  if (l < 4) { w->sp_has[l] = w->slow[l]; w->eb_has[l] = 0u; }
  __syncwarp();
  if (w->net) {
    const int nEW = (c.E + 31) >> 5;
    for (int i = l; i < nEW; i += 32) {
      for (unsigned m = c.w->edgebad[i]; m; m &= m - 1) {
        const int e = 32 * i + __ffs(m) - 1;
        for (int u = e * c.h; u < (e + 1) * c.h; ++u) {
          const int ch = __ldg(c.inv + u) >> 7;
          atomicOr(&w->slow[ch >> 5], 1u << (ch & 31));
          atomicOr(&w->eb_has[ch >> 5], 1u << (ch & 31));
        }
      }
    }
  }
  __syncwarp();
}

struct WStats {
  unsigned long long steps, retries, fp64, invalid, feas, scan_a, scan_b;
};

// Registers of the request a warp is scheduling.
struct WReq {
  int r, c0, nC, v0, nV, P, p;
  int cmin, cmax, rmin, rmax, cpod;        // container `lane`
  bool hc, hv0, hv1;
  int bn0, bx0, bn1, bx1;                  // vlinks `lane` and `lane + 32`
  int pa0, pb0, pa1, pb1, path0, path1;    // endpoint pods, chosen paths
  int pcpu, pram;                          // demand of pod `lane`
};

__device__ __forceinline__ void emit_failed(const OutDev& O, const WReq& q, int lane, int status) {
  if (q.hc) { O.server[q.c0 + lane] = -1; O.cpu_a[q.c0 + lane] = 0; O.ram_a[q.c0 + lane] = 0; }
  if (q.hv0) { O.bw_a[q.v0 + lane] = 0; O.path[q.v0 + lane] = -1; }
  if (q.hv1) { O.bw_a[q.v0 + lane + 32] = 0; O.path[q.v0 + lane + 32] = -1; }
  if (lane == 0) O.status[q.r] = status;
}

// Fetch requests until one is accepted into the fast path (returns false when the batch
// is exhausted).  Oversized requests are deferred; invalid ones are emitted with -1.
template <typename LT>
__device__ bool acquire(WCtx<LT>& c, const ReqsDev& R, const OutDev& O, WReq& q, int* next, const int* order,
                        int* deferred, int* n_deferred, WStats& ws) {
  const int lane = c.lane;
  WScr* w = c.w;
  for (;;) {
    int r = 0;
    if (lane == 0) {
      r = atomicAdd(next, 1);
      if (r < R.n) r = order[r];
    }
    r = __shfl_sync(NACS_FULL, r, 0);
    if (r >= R.n) return false;
    q.r = r;
    q.c0 = R.coff[r];
    q.nC = R.coff[r + 1] - q.c0;
    q.v0 = R.voff[r];
    q.nV = R.voff[r + 1] - q.v0;
    if (q.nC > WC || q.nV > WV) {
      if (lane == 0) deferred[atomicAdd(n_deferred, 1)] = r;
      continue;
    }
    q.hc = lane < q.nC;
    q.cmin = q.cmax = q.rmin = q.rmax = 1;
    q.cpod = 0;
    if (q.hc) {
      q.cmin = R.cpu_min[q.c0 + lane]; q.cmax = R.cpu_max[q.c0 + lane];
      q.rmin = R.ram_min[q.c0 + lane]; q.rmax = R.ram_max[q.c0 + lane];
      q.cpod = R.pod_of[q.c0 + lane];
    }
    q.hv0 = lane < q.nV;
    q.hv1 = lane + 32 < q.nV;
    int s0 = 0, d0 = 1, s1 = 0, d1 = 1;
    q.bn0 = q.bx0 = q.bn1 = q.bx1 = 1;
    if (q.hv0) { s0 = R.src[q.v0 + lane]; d0 = R.dst[q.v0 + lane]; q.bn0 = R.bw_min[q.v0 + lane]; q.bx0 = R.bw_max[q.v0 + lane]; }
    if (q.hv1) {
      s1 = R.src[q.v0 + lane + 32]; d1 = R.dst[q.v0 + lane + 32];
      q.bn1 = R.bw_min[q.v0 + lane + 32]; q.bx1 = R.bw_max[q.v0 + lane + 32];
    }
    // validation (R24), in registers
    const int nC = q.nC;
    bool bad = q.hc && (q.cmin <= 0 || q.rmin <= 0 || q.cmin > q.cmax || q.rmin > q.rmax || q.cpod < 0 || q.cpod >= nC);
    bad |= q.hv0 && (s0 < 0 || s0 >= nC || d0 < 0 || d0 >= nC || s0 == d0 || q.bn0 <= 0 || q.bn0 > q.bx0);
    bad |= q.hv1 && (s1 < 0 || s1 >= nC || d1 < 0 || d1 >= nC || s1 == d1 || q.bn1 <= 0 || q.bn1 > q.bx1);
    unsigned used = __reduce_or_sync(NACS_FULL, q.hc && q.cpod >= 0 && q.cpod < 32 ? (1u << q.cpod) : 0u);
    int maxp = (int)__reduce_max_sync(NACS_FULL, q.hc && q.cpod >= 0 ? (unsigned)q.cpod : 0u);
    bool invalid = __any_sync(NACS_FULL, bad) || nC <= 0 || maxp >= 32 ||
                   used != (maxp == 31 ? 0xffffffffu : ((1u << (maxp + 1)) - 1u));
    if (invalid) {
      emit_failed(O, q, lane, -1);
      if (lane == 0) ws.invalid += 1;
      continue;
    }
    q.P = maxp + 1;
    q.p = 0;
    q.pcpu = q.pram = 0;
    for (int i = 0; i < nC; ++i) {
      int pd = __shfl_sync(NACS_FULL, q.cpod, i);
      int cm = __shfl_sync(NACS_FULL, q.cmin, i);
      int rm = __shfl_sync(NACS_FULL, q.rmin, i);
      if (lane == pd) { q.pcpu += cm; q.pram += rm; }
    }
    q.pa0 = __shfl_sync(NACS_FULL, q.cpod, s0 & 31);
    q.pb0 = __shfl_sync(NACS_FULL, q.cpod, d0 & 31);
    q.pa1 = __shfl_sync(NACS_FULL, q.cpod, s1 & 31);
    q.pb1 = __shfl_sync(NACS_FULL, q.cpod, d1 & 31);
    q.path0 = q.path1 = -1;
    w->pod_srv[lane] = -1;
    if (lane == 0) { w->nos = 0; w->nol = 0; }
    for (int i = lane; i < c.nDW; i += 32) c.w->dirty[i] = 0u;
    __syncwarp();
    return true;
  }
}

// a1/a2: flows of pod q.p to placed peers (R17), fabric tables, flow-server feasibility.
template <typename LT>
__device__ void prepare_step(WCtx<LT>& c, WReq& q, StepP& sp) {
  WScr* w = c.w;
  const int lane = c.lane, p = q.p;
  int ov0 = -1, ov1 = -1;
  if (q.hv0) {
    int other = (q.pa0 == p && q.pb0 != p) ? q.pb0 : ((q.pb0 == p && q.pa0 != p) ? q.pa0 : -1);
    if (other >= 0) ov0 = w->pod_srv[other];
  }
  if (q.hv1) {
    int other = (q.pa1 == p && q.pb1 != p) ? q.pb1 : ((q.pb1 == p && q.pa1 != p) ? q.pa1 : -1);
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
    int D = (int)__reduce_add_sync(NACS_FULL, (mine0 ? (unsigned)q.bn0 : 0u) + (mine1 ? (unsigned)q.bn1 : 0u));
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
  const bool net = c.o.path_filter && nflow > 0;
  if (net) wfabric(c);
  bool Gl = true;
  if (lane < nflow) {
    int v = w->fv[lane], D = w->fD[lane];
    int av = acc_val(c, v);
    Gl = av >= D;
    bool fk = av >= sumD - D;
    for (int f2 = 0; f2 < nflow; ++f2)
      if (f2 != lane && acc_val(c, w->fv[f2]) < w->fD[f2]) fk = false;
    if (net && ebad(c, (unsigned)v)) fk = false;
    w->fok[lane] = fk;
  }
  const bool G = __all_sync(NACS_FULL, Gl);
  const int dc = __shfl_sync(NACS_FULL, q.pcpu, p), dr = __shfl_sync(NACS_FULL, q.pram, p);
  sp.dc = dc;
  sp.dr = dr;
  sp.dcp = (net && !G) ? INT_MAX : dc;
  sp.walk = false;
  sp.f0c = sp.f0r = INT_MIN;
  sp.tc = sp.dcp;
  sp.tr = dr;
  sp.sumDp = net ? sumD : INT_MIN;
  sp.net = net;
  sp.pf = c.o.path_filter != 0;
  sp.h4 = (c.h & 3) == 0;
  if (lane == 0) { w->sumD = sumD; w->net = net; }
  __syncwarp();
}

// a8: commit the chosen server.  Returns 0 ok, 1 routing failed (R18), 2 overlay full.
// Warp-cooperative: every lane runs the same control flow, lane 0 writes.
template <typename LT>
__device__ int commit_step(WCtx<LT>& c, WReq& q, const StepP& sp, int best, int best_pos) {
  WScr* w = c.w;
  const int lane = c.lane;
  const int nos0 = w->nos;
  c.ulog_n = 0;
  int fail = 0;
  {
    int s = w_slot(c, best);
    int cu = s >= 0 ? w->os_cpu[s] : c.snap[tile_idx(best_pos, 0)];
    int ru = s >= 0 ? w->os_ram[s] : c.snap[tile_idx(best_pos, 1)];
    int qu = s >= 0 ? w->os_acc[s] : c.snap[tile_idx(best_pos, 3)];
    if (!w_set_server(c, best, best_pos, cu - sp.dc, ru - sp.dr, 1, qu)) fail = 2;
  }
  const int nflow = w->nflow;
  for (int fi = 0; fi < nflow && !fail; ++fi) {
    const int v = w->fv[fi], D = w->fD[fi];
    if (v == best) {
      if (lane == 0) w->fpath[fi] = -1;
      __syncwarp();
      continue;
    }
    const int2 wp = wpath(c, best, v);
    const int su = w_slot(c, best), sv = w_slot(c, v);
    const int au = w->os_acc[su];
    const int pv = sv >= 0 ? w->os_pos[sv] : __ldg(c.inv + v);
    const int av = sv >= 0 ? w->os_acc[sv] : c.snap[tile_idx(pv, 3)];
    if (min(min(au, av), wp.y) < D) {
      fail = 1;
      break;
    }
    bool ok = w_set_server(c, best, best_pos, w->os_cpu[su], w->os_ram[su], w->os_act[su], au - D);
    const int cv = sv >= 0 ? w->os_cpu[sv] : c.snap[tile_idx(pv, 0)];
    const int rv = sv >= 0 ? w->os_ram[sv] : c.snap[tile_idx(pv, 1)];
    const int tv = sv >= 0 ? w->os_act[sv] : (c.snap[tile_idx(pv, 2)] & 1);
    ok = ok && w_set_server(c, v, pv, cv, rv, tv, av - D);
    int fid[4];
    const int m = path_fids(c, best, v, wp.x, fid);
    for (int t = 0; t < m && ok; ++t) ok = w_add_link(c, fid[t], -D);
    if (!ok) fail = 2;
    if (lane == 0) w->fpath[fi] = wp.x;
    __syncwarp();
  }
  if (fail == 1) {
    w_undo(c, nos0);
    if (lane == 0) {
      if (w->nex < WX) { w->ex[w->nex] = best; w->ex_pos[w->nex] = best_pos; }
      w->nex += 1;
    }
  }
  if (fail == 0) {
    const int p = q.p;
    if (lane == 0) w->pod_srv[p] = best;
    __syncwarp();
    if (q.hv0) {
      int other = (q.pa0 == p && q.pb0 < p) ? q.pb0 : ((q.pb0 == p && q.pa0 < p) ? q.pa0 : -1);
      if (other >= 0) {
        int v = w->pod_srv[other];
        for (int i = 0; i < nflow; ++i) if (w->fv[i] == v) q.path0 = w->fpath[i];
      }
    }
    if (q.hv1) {
      int other = (q.pa1 == p && q.pb1 < p) ? q.pb1 : ((q.pb1 == p && q.pa1 < p) ? q.pa1 : -1);
      if (other >= 0) {
        int v = w->pod_srv[other];
        for (int i = 0; i < nflow; ++i) if (w->fv[i] == v) q.path1 = w->fpath[i];
      }
    }
  }
  __syncwarp();
  return fail;
}

// a9: top-up (R19) in container order then vlink order; emit M_c, M_ec, c^a, bw^a.
// Warp-cooperative like commit_step.
template <typename LT>
__device__ void finish_request(WCtx<LT>& c, const WReq& q, const OutDev& O) {
  WScr* w = c.w;
  const int lane = c.lane;
  // R19 containers, in container order: greedy per server = clamp of prefix sums.  Lane i
  // holds container i; with P = the extras wanted by the earlier containers on its server,
  // it gets min(P + x, R) - min(P, R) of the server's residual R.
  int my_ec = 0, my_er = 0;
  {
    const bool hc = lane < q.nC;
    const int s = hc ? os_slot(c, w->pod_srv[q.cpod]) : -1;  // a placed server is always overlaid
    const int xc = q.cmax - q.cmin, xr = q.rmax - q.rmin;
    if (hc) { w->dem[lane] = xc; w->dem[32 + lane] = xr; }
    const unsigned peers = __match_any_sync(NACS_FULL, s) & __ballot_sync(NACS_FULL, hc);
    __syncwarp();
    if (hc) {
      int pc = 0, pr = 0;
      for (unsigned m = peers & ((1u << lane) - 1u); m; m &= m - 1) {
        const int j = __ffs(m) - 1;
        pc += w->dem[j];
        pr += w->dem[32 + j];
      }
      const int Rc = w->os_cpu[s], Rr = w->os_ram[s];
      my_ec = min(pc + xc, Rc) - min(pc, Rc);
      my_er = min(pr + xr, Rr) - min(pr, Rr);
      if (lane == 31 - __clz(peers)) {  // the server's last container writes its residual
        w->os_cpu[s] = Rc - min(pc + xc, Rc);
        w->os_ram[s] = Rr - min(pr + xr, Rr);
      }
    }
    __syncwarp();
  }
  // R19 vlinks, in vlink order.  When no access link or fabric link is asked for more than
  // its residual by all the vlinks together, every vlink gets its whole extra and the
  // greedy order cannot matter: apply the sums in parallel.  Otherwise the sequential loop.
  int my_bw0 = 0, my_bw1 = 0;
  bool par = true;
  {
    int* dem_l = w->dem;        // [WOL] per overlay link position
    int* dem_s = w->dem + WOL;  // [WOS] per overlay server slot (its access link)
    for (int i = lane; i < WOL + WOS; i += 32) w->dem[i] = 0;
    __syncwarp();
#pragma unroll
    for (int hv = 0; hv < 2; ++hv) {
      const bool has = hv ? q.hv1 : q.hv0;
      if (!has) continue;
      const int us = w->pod_srv[hv ? q.pa1 : q.pa0], ud = w->pod_srv[hv ? q.pb1 : q.pb0];
      const int want = (hv ? q.bx1 - q.bn1 : q.bx0 - q.bn0);
      if (us == ud || want == 0) continue;
      atomicAdd(&dem_s[os_slot(c, us)], want);
      atomicAdd(&dem_s[os_slot(c, ud)], want);
      int fid[4];
      const int m = path_fids(c, us, ud, hv ? q.path1 : q.path0, fid);
      for (int t = 0; t < m; ++t) {
        const int p = ol_find(w, fid[t]);  // a reserved path's links are in the overlay
        if (p < 0) par = false;
        else atomicAdd(&dem_l[p], want);
      }
    }
    __syncwarp();
    for (int i = lane; i < w->nos; i += 32) par &= dem_s[i] <= w->os_acc[i];
    for (int i = lane; i < w->nol; i += 32) par &= dem_l[i] <= w->ol_val[i];
    par = __all_sync(NACS_FULL, par);
    if (par) {
      for (int i = lane; i < w->nos; i += 32) w->os_acc[i] -= dem_s[i];
      for (int i = lane; i < w->nol; i += 32) w->ol_val[i] -= dem_l[i];
      my_bw0 = q.bx0;
      my_bw1 = q.bx1;
    }
    __syncwarp();
  }
  for (int e = 0; e < (par ? 0 : q.nV); ++e) {
    const int src_lane = e & 31;
    const bool hi = e >= 32;
    const int es = __shfl_sync(NACS_FULL, hi ? q.pa1 : q.pa0, src_lane);
    const int ed = __shfl_sync(NACS_FULL, hi ? q.pb1 : q.pb0, src_lane);
    const int bmin = __shfl_sync(NACS_FULL, hi ? q.bn1 : q.bn0, src_lane);
    const int bmax = __shfl_sync(NACS_FULL, hi ? q.bx1 : q.bx0, src_lane);
    const int pid = __shfl_sync(NACS_FULL, hi ? q.path1 : q.path0, src_lane);
    const int us = w->pod_srv[es], ud = w->pod_srv[ed];
    int bw = bmax;
    if (us != ud) {
      const int ss = w_slot(c, us), sd = w_slot(c, ud);
      int fid[4];
      const int m = path_fids(c, us, ud, pid, fid);
      int resid = min(w->os_acc[ss], w->os_acc[sd]);
      for (int t = 0; t < m; ++t) resid = min(resid, fab_val(c, fid[t]));
      const int extra = min(bmax - bmin, resid);
      if (extra) {
        __syncwarp();
        if (lane == 0) { w->os_acc[ss] -= extra; w->os_acc[sd] -= extra; }
        __syncwarp();
        for (int t = 0; t < m; ++t) w_add_link(c, fid[t], -extra, false);
      }
      bw = bmin + extra;
    }
    if (lane == src_lane) { if (hi) my_bw1 = bw; else my_bw0 = bw; }
  }
  if (q.hc) {
    O.server[q.c0 + lane] = w->pod_srv[q.cpod];
    O.cpu_a[q.c0 + lane] = q.cmin + my_ec;
    O.ram_a[q.c0 + lane] = q.rmin + my_er;
  }
  if (q.hv0) {
    const bool intra = w->pod_srv[q.pa0] == w->pod_srv[q.pb0];
    O.bw_a[q.v0 + lane] = my_bw0;
    O.path[q.v0 + lane] = intra ? -1 : q.path0;
  }
  if (q.hv1) {
    const bool intra = w->pod_srv[q.pa1] == w->pod_srv[q.pb1];
    O.bw_a[q.v0 + lane + 32] = my_bw1;
    O.path[q.v0 + lane + 32] = intra ? -1 : q.path1;
  }
  if (lane == 0) O.status[q.r] = 1;
  __syncwarp();
}

// Named barrier over the nt threads of one warp group (id >= 1; 0 is __syncthreads).
__device__ __forceinline__ void group_sync(int id, int nt) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nt) : "memory");
}
__device__ __forceinline__ bool group_sync_and(int id, int nt, bool p) {
  int r;
  asm volatile(
      "{\n .reg .pred a, b;\n setp.ne.u32 a, %1, 0;\n bar.red.and.pred b, %2, %3, a;\n selp.u32 %0, 1, 0, b;\n}"
      : "=r"(r)
      : "r"((int)p), "r"(id), "r"(nt)
      : "memory");
  return r != 0;
}

// The warps of a CTA advance in lockstep phases (prepare | pass A | pass B | commit), each
// on its own request, so that all warps run the same loop at the same time (one copy of
// the hot code in the instruction caches); within a phase no warp waits for another.
template <typename LT, bool RO>  // RO: R25 rank-once instantiation
__global__ void __launch_bounds__(NACS_WARP_THREADS, 1) k_batch_warp(Geo g, Opt o, const int* __restrict__ state,
                                                       const int* __restrict__ lay, ReqsDev R, OutDev O,
                                                       int4* ulog_all, int* next, const int* order, int* deferred,
                                                       int* n_deferred, unsigned long long* stats, int group,
                                                       int sync_mask) {
  extern __shared__ __align__(16) unsigned char dyn[];
  const int n = g.n, h = g.h, k = g.k, E = g.E;
  const int npad = (n + 127) & ~127, nch = npad >> 7;
  // ---- a0: shared snapshot (read-only for the whole kernel): the chunk layout of the
  // criteria and the chunk table (k_warp_layout), the fabric links in switch order
  // per-warp scratch first (a compile-time stride), then the snapshot
  int* ssnap = reinterpret_cast<int*>(dyn + sizeof(WScr) * WWARPS);
  ChunkT* stab = reinterpret_cast<ChunkT*>(ssnap + 4 * npad);
  LT* sfab = reinterpret_cast<LT*>(stab + nch);
  const int nfab = E * h + k * h * h;
  const int nDW = (E + k * h + 31) >> 5;
  __shared__ __align__(8) unsigned long long mbar;
  __shared__ int s_fabmin;
  // criteria tiles and chunk table are contiguous in `lay` and in shared memory: TMA bulk
  const unsigned bytes = 16u * (unsigned)npad + (unsigned)sizeof(ChunkT) * (unsigned)nch;
  if (threadIdx.x == 0) {
    const unsigned mb = smem_addr(&mbar), chunk = 32768;
    s_fabmin = INT_MAX;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
    for (unsigned o2 = 0; o2 < bytes; o2 += chunk) {
      const unsigned sz = bytes - o2 < chunk ? bytes - o2 : chunk;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_addr(ssnap) + o2),
                   "l"(reinterpret_cast<const unsigned char*>(lay + LAY_PST) + o2), "r"(sz), "r"(mb)
                   : "memory");
    }
  }
  __syncthreads();
  {
    int m = INT_MAX;
    for (int i = threadIdx.x; i < nfab; i += blockDim.x) {
      const int v = __ldg(state + 4 * n + i);
      sfab[i] = (LT)v;
      m = min(m, v);
    }
    m = __reduce_min_sync(NACS_FULL, m);
    if ((threadIdx.x & 31) == 0) atomicMin(&s_fabmin, m);
  }
  __syncthreads();
  {
    const unsigned mb = smem_addr(&mbar);
    asm volatile(
        "{\n .reg .pred P1;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
        " @!P1 bra WAIT_%=;\n}" ::"r"(mb)
        : "memory");
  }

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // warp groups advance in lockstep independently (named barrier 1 + group index)
  const int nwarps = blockDim.x >> 5, gid = warp / group;
  const int bar_id = 1 + gid, bar_nt = 32 * min(group, nwarps - gid * group);
  WCtx<LT> c;
  c.k = k; c.h = h; c.n = n; c.npad = npad; c.E = E; c.nfabea = E * h;
  c.magic = g.magic_h;
  c.snap = ssnap;
  c.ctab = stab;
  c.inv = lay + LAY_PST + 4 * npad + 16 * nch;
  c.nch = nch;
  c.a_snap = smem_addr(ssnap) + 16u * lane;
  c.fab = sfab;
  c.w = reinterpret_cast<WScr*>(dyn) + warp;
  c.nDW = nDW;
  c.fabmin = s_fabmin;
  c.ulog = ulog_all + ((size_t)blockIdx.x * (blockDim.x >> 5) + warp) * WLOG;
  c.ulog_n = 0;
  c.lane = lane;
  c.o = o;
  WScr* w = c.w;
  const double wd[4] = {o.wd[0], o.wd[1], o.wd[2], o.wd[3]};
  WStats ws = {0, 0, 0, 0, 0, 0, 0};
  WReq q;
  q.r = -1;
  StepP sp;
  TopsisP tp;
  bool active = false, done = false, prep = false;
  int best = -1, best_pos = -1;

  for (;;) {
    // ---- phase P: acquire a request; flows and fabric tables of its pod step
    if (!active && !done) {
      active = acquire(c, R, O, q, next, order, deferred, n_deferred, ws);
      done = !active;
      prep = active;
    }
    if (active && prep) {
      prepare_step(c, q, sp);
      prep = false;
    }
    if (active) build_specials(c);
    if (group_sync_and(bar_id, bar_nt, done)) break;
    // ---- phase A (a3 + a4): filter and statistics
    bool stepping = active;
    const bool walk = RO && q.p > 0;  // R25: later pod steps walk the first step's order
    if (stepping && walk) {
      sp.walk = true;
      sp.f0c = w->dc0;
      sp.f0r = w->dr0;
      sp.tc = max(sp.dcp, sp.f0c);
      sp.tr = max(sp.dr, sp.f0r);
      pass_a_walk(c, sp);
      ws.steps += 1;
      tp = w->tp0;
    } else if (stepping) {
      AccA acc = {0, 0, UINT_MAX, UINT_MAX, UINT_MAX, 0u, 0u, 0u, 0ull, 0ull, 0ull};
      pass_a(c, sp, acc, ws.scan_a);
      const int nf = (int)__reduce_add_sync(NACS_FULL, (unsigned)acc.nf);
      ws.steps += 1;
      ws.feas += (unsigned long long)nf;
      if (nf == 0) {  // R20: reject the whole request
        emit_failed(O, q, lane, 0);
        active = false;
        stepping = false;
      } else {
        const int nact = (int)__reduce_add_sync(NACS_FULL, (unsigned)acc.nact);
        tp.mn[0] = (int)__reduce_min_sync(NACS_FULL, acc.mn0); tp.mx[0] = (int)__reduce_max_sync(NACS_FULL, acc.mx0);
        tp.mn[1] = (int)__reduce_min_sync(NACS_FULL, acc.mn1); tp.mx[1] = (int)__reduce_max_sync(NACS_FULL, acc.mx1);
        tp.mn[3] = (int)__reduce_min_sync(NACS_FULL, acc.mn3); tp.mx[3] = (int)__reduce_max_sync(NACS_FULL, acc.mx3);
        tp.mn[2] = nact == nf ? 1 : 0;
        tp.mx[2] = nact > 0 ? 1 : 0;
        unsigned long long sq[4] = {warp_sum_u64(acc.q0), warp_sum_u64(acc.q1), (unsigned long long)nact,
                                    warp_sum_u64(acc.q3)};
        topsis_params(tp, wd, sq);
        if (RO && lane == 0) {  // the first pod step: keep its order's parameters
          w->tp0 = tp;
          w->dc0 = sp.dc;
          w->dr0 = sp.dr;
        }
        __syncwarp();
      }
    }
    if (sync_mask & 1) group_sync(bar_id, bar_nt);
    // ---- phase B (a5T + a7): closeness, argmax (lowest index), FP64 near-tie re-decision
    if (stepping) {
      const float INF = __int_as_float(0x7f800000);
      AccB bb = {INF, INF, -1, -1};
      pass_b(c, sp, tp, bb, ws.scan_b);
      // smallest q (positive floats order like their bit patterns), lowest index on ties
      const unsigned key1 = __float_as_uint(bb.b1);
      const unsigned m1 = __reduce_min_sync(NACS_FULL, key1);
      best = (int)__reduce_min_sync(NACS_FULL, key1 == m1 ? (unsigned)bb.i1 : UINT_MAX);
      const bool winner = key1 == m1 && bb.i1 == best;
      {
        const unsigned wl = __ballot_sync(NACS_FULL, winner);
        best_pos = __shfl_sync(NACS_FULL, bb.p1, wl ? __ffs(wl) - 1 : 0);
      }
      const unsigned m2 = __reduce_min_sync(NACS_FULL, winner ? __float_as_uint(bb.b2) : key1);
      const float q1 = __uint_as_float(m1), q2 = __uint_as_float(m2);
      if (o.exact64 || m2 == m1 || q2 - q1 <= kTopsisDeltaQ * q1) {  // R14: FP64 near-tie re-decision
        const float thr = o.exact64 ? INF : q1 * (1.0f + 2.0f * kTopsisDeltaQ);
        double bv = -DBL_MAX;
        int bj = -1, bp = -1;
        scan_fp64(c, sp, tp, thr, bv, bj, bp);
        const int mine = bj;
        warp_argmax64(bv, bj);
        best = bj;
        const unsigned wl = __ballot_sync(NACS_FULL, mine == bj && bj >= 0);
        best_pos = __shfl_sync(NACS_FULL, bp, wl ? __ffs(wl) - 1 : 0);
        ws.fp64 += 1;
      }
      if (best < 0) {  // R25: no server of the first step's order is admitted (R20)
        emit_failed(O, q, lane, 0);
        active = false;
        stepping = false;
      }
    }
    if (sync_mask & 2) group_sync(bar_id, bar_nt);
    // ---- phase C (a8, a9): commit; next pod, retry (R18), or request end
    if (stepping) {
      int fail = commit_step(c, q, sp, best, best_pos);
      if (fail == 1) {
        ws.retries += 1;
        if (w->nex > WX || w->nos + w->nex > WSP) fail = 2;
      }
      if (fail == 2) {  // overlay full: the CTA kernel takes the request
        if (lane == 0) deferred[atomicAdd(n_deferred, 1)] = q.r;
        active = false;
      } else if (fail == 0) {
        q.p += 1;
        if (q.p == q.P) {
          finish_request(c, q, O);
          active = false;
        } else {
          prep = true;
        }
      }
    }
  }
  if (lane == 0) {
    if (ws.steps) atomicAdd(&stats[ST_POD_STEPS], ws.steps);
    if (ws.retries) atomicAdd(&stats[ST_RETRIES], ws.retries);
    if (ws.fp64) atomicAdd(&stats[ST_FP64], ws.fp64);
    if (ws.invalid) atomicAdd(&stats[ST_INVALID], ws.invalid);
    if (ws.feas) atomicAdd(&stats[ST_FEAS], ws.feas);
    if (ws.scan_a) atomicAdd(&stats[ST_SCAN_A], ws.scan_a);
    if (ws.scan_b) atomicAdd(&stats[ST_SCAN_B], ws.scan_b);
  }
}

// Largest requests first (LPT): a counting sort of request indices by descending container
// count, so that the last requests handed out are the shortest and the warps of a CTA
// run out of work together.  One CTA; the order within a size class is arbitrary (the
// requests are independent, R21, so results do not depend on it).
__device__ void order_lpt(const ReqsDev& R, int* order) {
  __shared__ int hist[MAXC + 2];
  __shared__ int base[MAXC + 2];
  for (int i = threadIdx.x; i < MAXC + 2; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  for (int r = threadIdx.x; r < R.n; r += blockDim.x) {
    int s = R.coff[r + 1] - R.coff[r];
    s = s < 0 ? 0 : (s > MAXC ? MAXC + 1 : s);
    atomicAdd(&hist[s], 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int s = MAXC + 1; s >= 0; --s) { base[s] = acc; acc += hist[s]; }
  }
  __syncthreads();
  for (int r = threadIdx.x; r < R.n; r += blockDim.x) {
    int s = R.coff[r + 1] - R.coff[r];
    s = s < 0 ? 0 : (s > MAXC ? MAXC + 1 : s);
    order[atomicAdd(&base[s], 1)] = r;
  }
}

// ------------------------------------------------------------ chunk layout ----
// The scans of k_batch_warp read the criteria in 128-slot chunks whose static boxes and
// aggregates let pass A take whole chunks at once and let pass B skip chunks by a bound.
// k_warp_layout orders the servers for tight boxes: first the "low" servers (some
// criterion below the largest pod demand of the batch, or the access link below a tenth
// of its capacity: the ones the thresholds actually cut) in 4 buckets of how low, then by
// f_u, then along a Z-order curve of (CPU, RAM, access link) quantised to 10 bits; ties by
// server index.
// The order changes only which servers share a chunk, never a result.

// Largest pod CPU / RAM demand (sum of c^min over a pod's containers) of the batch.
__global__ void k_pod_max(ReqsDev R, int* lay) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  int mc = 0, mr = 0;
  if (r < R.n) {
    const int c0 = R.coff[r], c1 = R.coff[r + 1];
    if (c1 > c0 && c1 - c0 <= WC) {
      for (int i = c0; i < c1; ++i) {
        const int p = R.pod_of[i];
        bool first = true;
        for (int j = c0; j < i; ++j) first &= R.pod_of[j] != p;
        if (!first) continue;
        long long sc = 0, sr = 0;
        for (int j = i; j < c1; ++j)
          if (R.pod_of[j] == p) { sc += R.cpu_min[j]; sr += R.ram_min[j]; }
        mc = (int)max((long long)mc, min(sc, (long long)INT_MAX));
        mr = (int)max((long long)mr, min(sr, (long long)INT_MAX));
      }
    }
  }
  mc = (int)__reduce_max_sync(NACS_FULL, (unsigned)mc);
  mr = (int)__reduce_max_sync(NACS_FULL, (unsigned)mr);
  if ((threadIdx.x & 31) == 0) {
    atomicMax(lay + 0, mc);
    atomicMax(lay + 1, mr);
  }
}

__device__ __forceinline__ unsigned spread3(unsigned x) {  // bits 0..9 -> every third bit
  x &= 0x3ffu;
  x = (x | (x << 16)) & 0x030000FFu;
  x = (x | (x << 8)) & 0x0300F00Fu;
  x = (x | (x << 4)) & 0x030C30C3u;
  x = (x | (x << 2)) & 0x09249249u;
  return x;
}
__device__ __forceinline__ unsigned quant10(int v, int vmax) {
  return (unsigned)(((long long)max(v, 0) << 10) / ((long long)vmax + 1));
}

// One CTA: sort the servers by layout key, write the criteria tiles, inv and the chunk table.
__device__ void warp_layout(const Geo& g, const int* __restrict__ state, int* lay) {
  extern __shared__ unsigned long long key[];
  __shared__ int smax[3];
  const int n = g.n, npad = (n + 127) & ~127, nch = npad >> 7;
  int P2 = 1;
  while (P2 < npad) P2 <<= 1;
  int* pst = lay + LAY_PST;
  ChunkT* tab = reinterpret_cast<ChunkT*>(pst + 4 * npad);
  int* inv = pst + 4 * npad + 16 * nch;
  const int* cpu = state;
  const int* ram = state + n;
  const int* act = state + 2 * n;
  const int* acc = state + 3 * n;
  if (threadIdx.x < 3) smax[threadIdx.x] = 0;
  __syncthreads();
  {
    int m0 = 0, m1 = 0, m2 = 0;
    for (int u = threadIdx.x; u < n; u += blockDim.x) {
      m0 = max(m0, cpu[u]);
      m1 = max(m1, ram[u]);
      m2 = max(m2, acc[u]);
    }
    m0 = (int)__reduce_max_sync(NACS_FULL, (unsigned)max(m0, 0));
    m1 = (int)__reduce_max_sync(NACS_FULL, (unsigned)max(m1, 0));
    m2 = (int)__reduce_max_sync(NACS_FULL, (unsigned)max(m2, 0));
    if ((threadIdx.x & 31) == 0) { atomicMax(&smax[0], m0); atomicMax(&smax[1], m1); atomicMax(&smax[2], m2); }
  }
  __syncthreads();
  const int Tc = lay[0], Tr = lay[1], Ta = max(1, g.link_cap / 10);
  for (int i = threadIdx.x; i < P2; i += blockDim.x) {
    unsigned long long kk = ~0ull;
    if (i < n) {
      const bool high = cpu[i] >= Tc && ram[i] >= Tr && acc[i] >= Ta;
      const unsigned z = (spread3(quant10(cpu[i], smax[0])) << 2) | (spread3(quant10(ram[i], smax[1])) << 1) |
                         spread3(quant10(acc[i], smax[2]));
      // low servers: by how low (4 buckets of min_c x_c / T_c), so that the low tiles of a
      // pod step are mostly wholly feasible or wholly cut
      unsigned bucket = 0;
      if (!high) {
        const float r = fminf(fminf((float)cpu[i] / (float)max(Tc, 1), (float)ram[i] / (float)max(Tr, 1)),
                              (float)acc[i] / (float)Ta);
        bucket = (unsigned)min(3, max(0, (int)(r * 4.0f)));
      }
      kk = ((unsigned long long)high << 63) | ((unsigned long long)bucket << 61) |
           ((unsigned long long)(act[i] & 1) << 60) | ((unsigned long long)z << 30) | (unsigned)i;
    }
    key[i] = kk;
  }
  __syncthreads();
  for (int kb = 2; kb <= P2; kb <<= 1) {
    for (int j = kb >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < P2; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const unsigned long long x = key[i], y = key[ixj];
          const bool up = (i & kb) == 0;
          if ((x > y) == up) { key[i] = y; key[ixj] = x; }
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < npad; i += blockDim.x) {
    const int t = i >> 7, l = i & 127;
    int* tile = pst + (t << 9);
    if (i < n) {
      const int u = (int)(key[i] & 0x3fffffffu);
      tile[l] = cpu[u];
      tile[128 + l] = ram[u];
      tile[256 + l] = (u << 1) | (act[u] & 1);
      tile[384 + l] = acc[u];
      inv[u] = i;
    } else {  // padding is never feasible (demands are > 0)
      tile[l] = -1;
      tile[128 + l] = -1;
      tile[256 + l] = 0;
      tile[384 + l] = 0;
    }
  }
  __syncthreads();
  // chunk table: one warp per chunk, 4 slots per lane
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int ch = warp; ch < nch; ch += blockDim.x >> 5) {
    int lo[3] = {INT_MAX, INT_MAX, INT_MAX}, hi[3] = {INT_MIN, INT_MIN, INT_MIN};
    int cnt = 0, nact = 0, am = 0;
    unsigned long long sq[3] = {0, 0, 0};
    for (int j = 0; j < 4; ++j) {
      const int i = (ch << 7) + 4 * lane + j;
      if (i >= n) continue;
      const int u = (int)(key[i] & 0x3fffffffu);
      const int x[3] = {cpu[u], ram[u], acc[u]};
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        lo[c] = min(lo[c], x[c]);
        hi[c] = max(hi[c], x[c]);
        sq[c] += (unsigned long long)((long long)x[c] * x[c]);
      }
      cnt += 1;
      nact += act[u] & 1;
      am |= 1 << (act[u] & 1);
    }
    ChunkT t;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      t.lo[c] = __reduce_min_sync(NACS_FULL, lo[c]);
      t.hi[c] = __reduce_max_sync(NACS_FULL, hi[c]);
      unsigned long long v = sq[c];
#pragma unroll
      for (int o2 = 16; o2 > 0; o2 >>= 1) v += __shfl_xor_sync(NACS_FULL, v, o2);
      t.sq[c] = v;
    }
    t.cnt = (int)__reduce_add_sync(NACS_FULL, (unsigned)cnt);
    t.nact = (int)__reduce_add_sync(NACS_FULL, (unsigned)nact);
    t.act = (int)__reduce_or_sync(NACS_FULL, (unsigned)am);
    t.pad = 0;
    if (lane == 0) tab[ch] = t;
  }
}

// ------------------------------------------------------------------- host ----
static size_t warp_snapshot_bytes(const Geo& g, bool u16) {
  size_t npad = (size_t)((g.n + 127) & ~127);
  size_t nfab = (size_t)g.E * g.h + (size_t)g.k * g.h * g.h;
  return 16 * npad + sizeof(ChunkT) * (npad >> 7) + (((u16 ? 2 : 4) * nfab + 15) & ~(size_t)15);
}
size_t warp_layout_ints(const Geo& g) {
  size_t npad = (size_t)((g.n + 127) & ~127);
  return LAY_PST + 4 * npad + 16 * (npad >> 7) + (size_t)g.n;
}

int warp_kernel_warps(const Geo& g) {
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  bool u16 = g.link_cap <= 65535;
  // dynamic shared memory: WWARPS per-warp scratch areas + the snapshot (+ static words)
  const size_t stat = sizeof(WScr) * WWARPS + 64;
  if (warp_snapshot_bytes(g, u16) + stat > (size_t)optin || ((g.n + 127) >> 7) > WCH) return 0;
  if (g.E > 32 * WEW || g.E + g.k * g.h > 32 * WDW || g.k > 64) return 0;
  return NACS_WARP_THREADS / 32;
}

size_t warp_ulog_entries(int grid, int warps) { return (size_t)grid * warps * WLOG; }

// The chunk layout (CTA 0) and the largest-first request order (CTA 1) are independent:
// one launch of two CTAs runs them side by side (they were two one-CTA launches in a row).
__global__ void __launch_bounds__(1024) k_layout_order(Geo g, const int* __restrict__ state, int* lay, ReqsDev R,
                                                       int* order) {
  if (blockIdx.x == 0) warp_layout(g, state, lay);
  else order_lpt(R, order);
}

cudaError_t launch_batch_warp(const Geo& g, const Opt& o, const int* d_state, int* lay, const ReqsDev& R,
                              const OutDev& O, int4* ulog, int* next, int* order, int* deferred, int* n_deferred,
                              unsigned long long* stats, int grid, int warps, cudaStream_t st) {
  bool u16 = g.link_cap <= 65535;
  cudaError_t e = cudaMemsetAsync(lay, 0, 4 * sizeof(int), st);
  if (e != cudaSuccess) return e;
  if (R.n > 0) k_pod_max<<<(R.n + 255) / 256, 256, 0, st>>>(R, lay);
  {
    const int npad = (g.n + 127) & ~127;
    int P2 = 1;
    while (P2 < npad) P2 <<= 1;
    const size_t lsm = sizeof(unsigned long long) * (size_t)P2;
    cudaFuncSetAttribute(k_layout_order, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lsm);
    k_layout_order<<<2, 1024, lsm, st>>>(g, d_state, lay, R, order);
  }
  // lockstep group size and the optional barriers before phases B / C (A/B on one box, C4,
  // NACS_WARP_GROUP / NACS_WARP_SYNC override): per-pod, the whole CTA in lockstep with a
  // barrier before the commit only, 12.74 ms (groups of 8 with both barriers 13.43 ms, 16 with
  // none 13.20, 16 with both 13.05); rank-once keeps groups of 8 with both (6.60 vs 6.82 ms)
  static const char* eg = getenv("NACS_WARP_GROUP");
  static const char* es = getenv("NACS_WARP_SYNC");
  int group = eg ? atoi(eg) : (o.rank_once ? 8 : 16);
  group = group < 1 ? 1 : (group > 16 ? 16 : group);
  const int sync_mask = es ? atoi(es) : (o.rank_once ? 3 : 2);
  size_t smem = warp_snapshot_bytes(g, u16) + sizeof(WScr) * WWARPS;
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<grid, warps * 32, smem, st>>>(g, o, d_state, lay, R, O, ulog, next, order, deferred, n_deferred, stats,
                                         group, sync_mask);
  };
  if (u16) {
    if (o.rank_once) go(k_batch_warp<uint16_t, true>);
    else go(k_batch_warp<uint16_t, false>);
  } else {
    if (o.rank_once) go(k_batch_warp<int, true>);
    else go(k_batch_warp<int, false>);
  }
  return cudaGetLastError();
}

}  // namespace nacs
