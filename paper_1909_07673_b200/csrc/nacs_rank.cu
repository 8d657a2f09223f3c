// nacs_rank.cu — whole-GPU TOPSIS ranking of one pod step on one or many DC states
// (§8(d) "standalone nacs_rank_topsis on cold snapshots").
//
// One THREAD-BLOCK CLUSTER ranks one DC state: the C = ceil(n / 4096) CTAs of the cluster
// each own a slice of <= 4096 servers, held in registers for every pass.  Per state:
//   a2  fabric feasibility of the slice's edge switches for every flow (shared memory),
//   a3+a4 filter + exact integer statistics of the slice   -> DSMEM exchange
//   a5T FP32 closeness, scores/mask written, top-2 keys    -> DSMEM exchange
//   a7  argmax; near ties re-decided in FP64  -> DSMEM exchange.
// Every CTA of a cluster reduces the C partials the same way (exact integers, order-free
// top-2 merges), so all of them take the same decision without another round trip; one
// cluster barrier per state publishes that state's statistics and the previous state's keys
// (the decision of state i is taken while state i+1 is ranked).  A persistent grid of
// clusters walks the states (state b -> cluster b mod #clusters), so one call streams B
// states: the algorithmic traffic is 16 B read per server (cpu, ram, f_u, access link) plus
// the 4 B score (and 1 B mask) written.  Paper: TOPSIS P:365-375 (R12-R13), filter Eq. 4-7
// P:181-189 (R6), "parallel reduction" P:380.
//
// Two kernels:
//  * k_rank_occ (16-byte aligned states, no flows or exclusions — the streaming case and the
//    first pod step of every request): 256 threads x 16 servers, TWO CTAs of different
//    clusters per SM (one computes while the other waits at its barrier), rows by TMA
//    (cp.async.bulk) into a stage, scores out by TMA bulk stores, CTA statistics by
//    shared-memory atomics of 32-bit warp reductions.
//  * k_rank_many (everything else: flows, exclusions, n % 4 != 0): 512 threads x 8 servers,
//    one CTA per SM, rows by TMA (aligned) or plain loads, flows' fabric tables per slice.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdlib>
#include <cstring>
#include <climits>

#include "nacs_device.cuh"
#include "nacs_internal.h"

namespace cg = cooperative_groups;

namespace nacs {

namespace {

constexpr int RM_T = 512;            // threads per CTA
constexpr int RM_V = 8;              // servers per thread
constexpr int RM_S = RM_T * RM_V;    // servers per CTA (slice)
constexpr int RM_NW = RM_T / 32;
constexpr int RM_EW = RM_S / 32 + 2; // words of the slice's edge bitmap (h = 1: one edge per server)

struct WStats {  // one warp's partial statistics over its part of the slice (read over DSMEM)
  unsigned long long q[3];    // sums of squares of CPU, RAM, access link over its feasible servers
  int nf, nact;
  unsigned mn[3], mx[3];      // CPU, RAM, access link over its feasible servers
  unsigned vmax[4];           // largest value of every criterion over all its servers (R5 range check)
};
struct WKeys {  // one warp's FP32 top-2 keys (score bits << 32 | ~server)
  unsigned long long k1, k2;
};

__device__ __forceinline__ void ldv(const int* p, int (&x)[4]) {
  const int4 v = __ldcs(reinterpret_cast<const int4*>(p));
  x[0] = v.x; x[1] = v.y; x[2] = v.z; x[3] = v.w;
}
__device__ __forceinline__ void ldv(const int* p, int (&x)[2]) {
  const int2 v = __ldcs(reinterpret_cast<const int2*>(p));
  x[0] = v.x; x[1] = v.y;
}
__device__ __forceinline__ void stv(float* p, const float (&x)[4]) {
  __stcs(reinterpret_cast<float4*>(p), make_float4(x[0], x[1], x[2], x[3]));
}
__device__ __forceinline__ void stv(float* p, const float (&x)[2]) {
  __stcs(reinterpret_cast<float2*>(p), make_float2(x[0], x[1]));
}
__device__ __forceinline__ void stm(uint8_t* p, unsigned bits) {  // 4 flags -> 4 bytes
  *reinterpret_cast<unsigned*>(p) = (bits & 1u) | ((bits & 2u) << 7) | ((bits & 4u) << 14) | ((bits & 8u) << 21);
}
__device__ __forceinline__ void stm2(uint8_t* p, unsigned bits) {
  *reinterpret_cast<unsigned short*>(p) = (unsigned short)((bits & 1u) | ((bits & 2u) << 7));
}

}  // namespace

// Per-CTA shared state of k_rank_many.  Slots [2] alternate between consecutive states of
// the cluster (iteration parity): a CTA writes slot p of iteration i+2 only after the
// cluster barrier of iteration i+1, which every CTA reaches after its reads of iteration i.
struct RmShared {
  WStats ws[2][RM_NW];
  WKeys wk[2][RM_NW];
  TopsisP tp[2];                // the cluster's TOPSIS parameters of the state (warp 0 -> all threads)
  int NF[2], BAD[2], state[2];  // feasible count, range violation, state index of the slot
  double argv;                  // FP64 re-decision: this CTA's best (value, server)
  int argj;
  int best, amb;
  WStats rs[RM_NW];             // cluster reduction, stage 1: warp w combines warp w of every CTA
  WKeys rk[RM_NW];
  unsigned long long cnt[4];    // rank 0: states decided, feasible servers, FP64 decisions, invalid states
  unsigned edgebad[RM_EW];      // slice edge e (relative to the slice's first edge): some flow fails
  unsigned special[RM_S / 32];  // slice server: a flow server or an excluded server
  unsigned pm[MAXK];            // a2 scratch: per fat-tree pod, bit a = core route via agg a ok
  unsigned vm;                  // a2 scratch: the flow server's edge uplinks >= D
  int fv[MAXF], fD[MAXF];
  int fok[MAXF], fexcl[MAXF];
  int sumD, G;
};

struct RmThread {  // per-thread constants of k_rank_many
  int C, rank, tid, lane, warp, lo, hi, e_lo, e_hi;
  bool net;
};

template <int VW>
__device__ __forceinline__ void rm_load(const RankManyArgs& a, const RmThread& t, int b,
                                        int (&y)[RM_V / VW][4][VW]) {
  const int n = a.g.n;
  const int* sp = a.states + (long long)b * a.stride;
#pragma unroll
  for (int j = 0; j < RM_V / VW; ++j) {
    const int u0 = t.lo + VW * (t.tid + RM_T * j);
    if (u0 < t.hi) {
#pragma unroll
      for (int c = 0; c < 4; ++c) ldv(sp + c * n + u0, y[j][c]);
    } else {
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int v = 0; v < VW; ++v) y[j][c][v] = 0;
    }
  }
}

// a2 + flow servers + exclusions of state b into the slice's bitmaps (shared memory)
__device__ void rm_flows(const RankManyArgs& a, const RmThread& t, RmShared& sm, const int* st) {
  const Geo& g = a.g;
  const int n = g.n, tid = t.tid;
  for (int w = tid; w < RM_EW; w += RM_T) sm.edgebad[w] = 0u;
  for (int w = tid; w < RM_S / 32; w += RM_T) sm.special[w] = 0u;
  if (tid < a.nflow) {
    sm.fv[tid] = a.fv[tid];
    sm.fD[tid] = a.fD[tid];
    sm.fexcl[tid] = 0;
  }
  if (tid == 0) {
    int s = 0, G = 1;
    for (int f = 0; f < a.nflow; ++f) {
      s += a.fD[f];
      if (st[3 * n + a.fv[f]] < a.fD[f]) G = 0;
    }
    sm.sumD = s;
    sm.G = G;
  }
  __syncthreads();
  const int* EA = st + 4 * n;
  const int* AC = EA + g.E * g.h;
  if (t.net && t.lo < t.hi) {
    const int h = g.h;
    const int p_lo = (int)div_h((unsigned)t.e_lo, g.magic_h), p_hi = (int)div_h((unsigned)t.e_hi, g.magic_h);
    for (int f = 0; f < a.nflow; ++f) {
      const int v = sm.fv[f], D = sm.fD[f];
      const int ev = (int)div_h((unsigned)v, g.magic_h), pv = (int)div_h((unsigned)ev, g.magic_h);
      // pm[p] bit a: some core (a, b) joins pod p and pod pv with both links >= D
      for (int p = p_lo + tid; p <= p_hi; p += RM_T) sm.pm[p] = 0u;
      if (tid == 0) sm.vm = 0u;
      __syncthreads();
      for (int q = tid; q < (p_hi - p_lo + 1) * h; q += RM_T) {
        const int pr = (int)div_h((unsigned)q, g.magic_h), aa = q - pr * h, p = p_lo + pr;
        const int* r1 = AC + (p * h + aa) * h;
        const int* r2 = AC + (pv * h + aa) * h;
        bool ok = false;
        for (int bb = 0; bb < h && !ok; ++bb) ok = r1[bb] >= D && r2[bb] >= D;
        if (ok) atomicOr(&sm.pm[p], 1u << aa);
      }
      for (int aa = tid; aa < h; aa += RM_T)
        if (EA[ev * h + aa] >= D) atomicOr(&sm.vm, 1u << aa);
      __syncthreads();
      const unsigned vm = sm.vm;
      for (int e = t.e_lo + tid; e <= t.e_hi; e += RM_T) {
        if (e == ev) continue;  // same edge switch: access links only
        unsigned em = 0;
        for (int aa = 0; aa < h; ++aa) em |= (EA[e * h + aa] >= D ? 1u : 0u) << aa;
        const int pe = (int)div_h((unsigned)e, g.magic_h);
        const unsigned ok = pe == pv ? (em & vm) : (em & vm & sm.pm[pe]);
        if (!ok) atomicOr(&sm.edgebad[(e - t.e_lo) >> 5], 1u << ((e - t.e_lo) & 31));
      }
      __syncthreads();
    }
  }
  // flow servers (their own flow runs on the host bus, R17) and excluded servers (R18)
  if (tid < a.nflow) {
    const int f = tid, u = sm.fv[f];
    if (u >= t.lo && u < t.hi) {
      bool ok = st[3 * n + u] >= sm.sumD - sm.fD[f];
      for (int o = 0; o < a.nflow; ++o)
        if (o != f && st[3 * n + sm.fv[o]] < sm.fD[o]) ok = false;
      const int e = (int)div_h((unsigned)u, g.magic_h) - t.e_lo;
      if (t.net && ((sm.edgebad[e >> 5] >> (e & 31)) & 1u)) ok = false;
      sm.fok[f] = ok;
      atomicOr(&sm.special[(u - t.lo) >> 5], 1u << ((u - t.lo) & 31));
    }
  }
  __syncthreads();
  for (int i = tid; i < a.nex; i += RM_T) {
    const int u = a.ex[i];
    if (u >= t.lo && u < t.hi) atomicOr(&sm.special[(u - t.lo) >> 5], 1u << ((u - t.lo) & 31));
    for (int f = 0; f < a.nflow; ++f)
      if (sm.fv[f] == u) sm.fexcl[f] = 1;
  }
  __syncthreads();
}

// a3: feasibility of server u with values x (flows: bitmaps of rm_flows)
template <bool FLOWS>
__device__ __forceinline__ bool rm_feasible(const RankManyArgs& a, const RmThread& t, const RmShared& sm,
                                            int u, int x0, int x1, int x3) {
  bool k = x0 >= a.dc && x1 >= a.dr;  // demands > 0: padding (u >= hi, values 0) never passes
  if (FLOWS && u < t.hi) {
    const Geo& g = a.g;
    if (t.net) {
      const int e = (int)div_h((unsigned)u, g.magic_h) - t.e_lo;
      k = k && sm.G && x3 >= sm.sumD && !((sm.edgebad[e >> 5] >> (e & 31)) & 1u);
    }
    if ((sm.special[(u - t.lo) >> 5] >> ((u - t.lo) & 31)) & 1u) {
      int f = -1;
      for (int i = 0; i < a.nflow; ++i) if (sm.fv[i] == u) f = i;
      k = f >= 0 && !sm.fexcl[f] && x0 >= a.dc && x1 >= a.dr && (!a.path_filter || sm.fok[f]);
    }
  }
  return k;
}

// After a cluster barrier, every warp w: combine warp partial w of the C CTAs (lane r reads
// rank r over DSMEM) for slot p's statistics and, when `keys`, slot q's keys.  Exact integer
// reductions (any order); the top-2 merge is order-free too.
__device__ void rm_gather(const RankManyArgs& a, const RmThread& t, RmShared& sm, cg::cluster_group& cl, int p,
                          bool keys, int q) {
  const bool in = t.lane < t.C;
  const int r = in ? t.lane : 0;
  const WStats* w = cl.map_shared_rank(&sm.ws[p][t.warp], r);
  int nf = in ? w->nf : 0, nact = in ? w->nact : 0;
  unsigned mn0 = in ? w->mn[0] : UINT_MAX, mn1 = in ? w->mn[1] : UINT_MAX, mn3 = in ? w->mn[2] : UINT_MAX;
  unsigned mx0 = in ? w->mx[0] : 0, mx1 = in ? w->mx[1] : 0, mx3 = in ? w->mx[2] : 0;
  unsigned v0 = in ? w->vmax[0] : 0, v1 = in ? w->vmax[1] : 0, v2 = in ? w->vmax[2] : 0, v3 = in ? w->vmax[3] : 0;
  unsigned long long q0 = in ? w->q[0] : 0, q1 = in ? w->q[1] : 0, q3 = in ? w->q[2] : 0;
  unsigned long long k1 = 0, k2 = 0;
  if (keys && in) {
    const WKeys* kk = cl.map_shared_rank(&sm.wk[q][t.warp], r);
    k1 = kk->k1;
    k2 = kk->k2;
  }
  nf = (int)__reduce_add_sync(NACS_FULL, (unsigned)nf);
  nact = (int)__reduce_add_sync(NACS_FULL, (unsigned)nact);
  mn0 = __reduce_min_sync(NACS_FULL, mn0); mx0 = __reduce_max_sync(NACS_FULL, mx0);
  mn1 = __reduce_min_sync(NACS_FULL, mn1); mx1 = __reduce_max_sync(NACS_FULL, mx1);
  mn3 = __reduce_min_sync(NACS_FULL, mn3); mx3 = __reduce_max_sync(NACS_FULL, mx3);
  v0 = __reduce_max_sync(NACS_FULL, v0); v1 = __reduce_max_sync(NACS_FULL, v1);
  v2 = __reduce_max_sync(NACS_FULL, v2); v3 = __reduce_max_sync(NACS_FULL, v3);
  q0 = warp_sum_u64(q0);
  q1 = warp_sum_u64(q1);
  q3 = warp_sum_u64(q3);
  if (keys) warp_top2(k1, k2);
  if (t.lane == 0) {
    WStats& o = sm.rs[t.warp];
    o.nf = nf; o.nact = nact;
    o.mn[0] = mn0; o.mx[0] = mx0; o.mn[1] = mn1; o.mx[1] = mx1; o.mn[2] = mn3; o.mx[2] = mx3;
    o.vmax[0] = v0; o.vmax[1] = v1; o.vmax[2] = v2; o.vmax[3] = v3;
    o.q[0] = q0; o.q[1] = q1; o.q[2] = q3;
    sm.rk[t.warp].k1 = k1;
    sm.rk[t.warp].k2 = k2;
  }
}

// Warp 0 after rm_gather + __syncthreads: the TOPSIS parameters of slot p's state (R12-R13;
// lane c computes criterion c's FP64 norm and scale) and the R5 range check.
__device__ void rm_params(const RankManyArgs& a, const RmThread& t, RmShared& sm, int p) {
  const bool in = t.lane < RM_NW;
  const WStats& w = sm.rs[in ? t.lane : 0];
  int nf = in ? w.nf : 0, nact = in ? w.nact : 0;
  unsigned mn0 = in ? w.mn[0] : UINT_MAX, mn1 = in ? w.mn[1] : UINT_MAX, mn3 = in ? w.mn[2] : UINT_MAX;
  unsigned mx0 = in ? w.mx[0] : 0, mx1 = in ? w.mx[1] : 0, mx3 = in ? w.mx[2] : 0;
  unsigned v0 = in ? w.vmax[0] : 0, v1 = in ? w.vmax[1] : 0, v2 = in ? w.vmax[2] : 0, v3 = in ? w.vmax[3] : 0;
  unsigned long long q0 = in ? w.q[0] : 0, q1 = in ? w.q[1] : 0, q3 = in ? w.q[2] : 0;
  nf = (int)__reduce_add_sync(NACS_FULL, (unsigned)nf);
  nact = (int)__reduce_add_sync(NACS_FULL, (unsigned)nact);
  mn0 = __reduce_min_sync(NACS_FULL, mn0); mx0 = __reduce_max_sync(NACS_FULL, mx0);
  mn1 = __reduce_min_sync(NACS_FULL, mn1); mx1 = __reduce_max_sync(NACS_FULL, mx1);
  mn3 = __reduce_min_sync(NACS_FULL, mn3); mx3 = __reduce_max_sync(NACS_FULL, mx3);
  v0 = __reduce_max_sync(NACS_FULL, v0); v1 = __reduce_max_sync(NACS_FULL, v1);
  v2 = __reduce_max_sync(NACS_FULL, v2); v3 = __reduce_max_sync(NACS_FULL, v3);
  q0 = warp_sum_u64(q0);
  q1 = warp_sum_u64(q1);
  q3 = warp_sum_u64(q3);
  // ||x_c|| = sqrt(sum over F of x_c^2), exact integer sums; lane c: criterion c
  const int c = t.lane & 3;
  const unsigned long long sq = c == 0 ? q0 : c == 1 ? q1 : c == 2 ? (unsigned long long)nact : q3;
  const double N = sqrt((double)sq);
  const double sdc = N > 0 ? a.wd[c] / N : 0.0;
  double sd[4];
#pragma unroll
  for (int cc = 0; cc < 4; ++cc) sd[cc] = __shfl_sync(NACS_FULL, sdc, cc);
  if (t.lane == 0) {
    TopsisP& tp = sm.tp[p];
    const int mn[4] = {(int)mn0, (int)mn1, nact == nf ? 1 : 0, (int)mn3};  // f_u in {0,1}
    const int mx[4] = {(int)mx0, (int)mx1, nact > 0 ? 1 : 0, (int)mx3};
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
      tp.mn[cc] = mn[cc];
      tp.mx[cc] = mx[cc];
      tp.sd[cc] = sd[cc];
      tp.sf[cc] = (float)sd[cc];
      tp.s2p23[cc] = (float)sd[cc] * 8388608.0f;
      tp.mxb[cc] = 0x4B000000 + mx[cc];
      tp.mnb[cc] = 0x4B000000 - mn[cc];
    }
    const float q2 = __fmul_rn(tp.sf[2], tp.sf[2]);
    tp.p2sq[0] = mx[2] - 0 ? q2 : 0.f;
    tp.p2sq[1] = mx[2] - 1 ? q2 : 0.f;
    tp.m2sq[0] = 0 - mn[2] ? q2 : 0.f;
    tp.m2sq[1] = 1 - mn[2] ? q2 : 0.f;
    sm.NF[p] = nf;
    // R5: every value an exact FP32 integer in its range (device-pointer states are validated
    // here; a violation invalidates the state's result)
    sm.BAD[p] = v0 > (unsigned)a.g.cpu_cap || v1 > (unsigned)a.g.ram_cap || v2 > 1u || v3 > (unsigned)a.g.link_cap;
  }
}

// Warp 1 after rm_gather + __syncthreads: the argmax of slot q's state from the gathered keys,
// and whether the FP32 top-2 gap is ambiguous (<= 2^-17 -> FP64 re-decision).
__device__ void rm_keys(const RankManyArgs& a, const RmThread& t, RmShared& sm, int q) {
  unsigned long long k1 = t.lane < RM_NW ? sm.rk[t.lane].k1 : 0ull;
  unsigned long long k2 = t.lane < RM_NW ? sm.rk[t.lane].k2 : 0ull;
  warp_top2(k1, k2);
  if (t.lane == 0) {
    const float s1 = __uint_as_float((unsigned)(k1 >> 32));
    const float s2 = __uint_as_float((unsigned)(k2 >> 32));
    const bool live = sm.NF[q] > 0 && !sm.BAD[q];
    sm.best = k1 ? (int)(0xFFFFFFFFu - (unsigned)(k1 & 0xFFFFFFFFull)) : -1;
    sm.amb = live && k1 && (a.exact64 || (k2 != 0ull && s1 - s2 <= kTopsisDelta));
    sm.argv = (double)s1;
  }
}

// FP64 re-decision of a near tie (R14): this CTA's best FP64 candidate among the
// feasible servers of its slice whose FP32 closeness is >= thr; the state's rows are read
// again from global memory (rare: the registers hold other states by now).
template <bool FLOWS>
__device__ void rm_fp64_slice(const RankManyArgs& a, const RmThread& t, RmShared& sm, int b, const TopsisP& tp,
                              float thr) {
  const int n = a.g.n;
  const int* st = a.states + (long long)b * a.stride;
  if (FLOWS) rm_flows(a, t, sm, st);
  double bv = -DBL_MAX;
  int bj = -1;
  for (int u = t.lo + t.tid; u < t.hi; u += RM_T) {
    const int x0 = st[u], x1 = st[n + u], x2 = st[2 * n + u], x3 = st[3 * n + u];
    if (!rm_feasible<FLOWS>(a, t, sm, u, x0, x1, x3)) continue;
    if (topsis32(tp, x0, x1, x2, x3) < thr) continue;
    const double r = topsis64(tp, x0, x1, x2, x3);
    if (r > bv || (r == bv && u < bj)) { bv = r; bj = u; }
  }
  warp_argmax64(bv, bj);
  __shared__ double rd[RM_NW];
  __shared__ int rj[RM_NW];
  if (t.lane == 0) { rd[t.warp] = bv; rj[t.warp] = bj; }
  __syncthreads();
  if (t.warp == 0) {
    bv = t.lane < RM_NW ? rd[t.lane] : -DBL_MAX;
    bj = t.lane < RM_NW ? rj[t.lane] : -1;
    warp_argmax64(bv, bj);
    if (t.lane == 0) { sm.argv = bv; sm.argj = bj; }
  }
}

// Finish slot q's state after rm_keys: the FP64 re-decision when ambiguous (two more cluster
// barriers; every CTA computed the same keys, so all take the branch), then rank 0 writes.
template <bool FLOWS>
__device__ void rm_finish(const RankManyArgs& a, const RmThread& t, RmShared& sm, cg::cluster_group& cl, int q) {
  const bool amb = sm.amb;
  const int b = sm.state[q];
  if (amb) {
    const float thr = a.exact64 ? -1.0f : (float)sm.argv - 2.0f * kTopsisDelta;
    __syncthreads();
    rm_fp64_slice<FLOWS>(a, t, sm, b, sm.tp[q], thr);
    cl.sync();  // every CTA's FP64 candidate is visible
    if (t.warp == 0) {
      double bv = -DBL_MAX;
      int bj = -1;
      if (t.lane < t.C) {
        const double* v = cl.map_shared_rank(&sm.argv, t.lane);
        const int* j = cl.map_shared_rank(&sm.argj, t.lane);
        if (*j >= 0) { bv = *v; bj = *j; }
      }
      warp_argmax64(bv, bj);
      if (t.lane == 0) sm.best = bj;
    }
    cl.sync();  // nobody rewrites argv / argj before every CTA has read them
  }
  if (t.rank == 0 && t.tid == 0) {  // counters kept per CTA, flushed once at the end
    const int NF = sm.NF[q], BAD = sm.BAD[q];
    a.best[b] = BAD ? -2 : (NF > 0 ? sm.best : -1);
    sm.cnt[0] += 1;
    sm.cnt[1] += (unsigned long long)NF;
    sm.cnt[2] += amb ? 1 : 0;
    sm.cnt[3] += BAD ? 1 : 0;
  }
}

// One state (iteration i, slot p = i & 1): filter + statistics into the warp slots, ONE
// cluster barrier (it publishes this state's statistics and the previous state's keys), the
// cluster reductions (every warp, then warps 0 / 1), the previous state's decision,
// closeness + scores + this state's keys into the warp slots.
template <int VW, bool FLOWS>
__device__ __forceinline__ void rm_state(const RankManyArgs& a, const RmThread& t, RmShared& sm,
                                         cg::cluster_group& cl, int b, int i, const int (&x)[RM_V / VW][4][VW]) {
  constexpr int NJ = RM_V / VW;
  const int n = a.g.n;
  const int tid = t.tid, lane = t.lane, warp = t.warp, p = i & 1;
  if (FLOWS) rm_flows(a, t, sm, a.states + (long long)b * a.stride);
  // --------------------------------------------------- a3 + a4: filter, stats --
  unsigned okb = 0;  // bit j * VW + v: server feasible
  int nf = 0, nact = 0;
  unsigned mn0 = UINT_MAX, mn1 = UINT_MAX, mn3 = UINT_MAX, mx0 = 0, mx1 = 0, mx3 = 0;
  unsigned v0 = 0, v1 = 0, v2 = 0, v3 = 0;
  unsigned long long q0 = 0, q1 = 0, q3 = 0;
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    const int u0 = t.lo + VW * (tid + RM_T * j);
#pragma unroll
    for (int v = 0; v < VW; ++v) {
      const unsigned x0 = (unsigned)x[j][0][v], x1 = (unsigned)x[j][1][v], x2 = (unsigned)x[j][2][v],
                     x3 = (unsigned)x[j][3][v];
      v0 = max(v0, x0); v1 = max(v1, x1); v2 = max(v2, x2); v3 = max(v3, x3);
      const bool k = rm_feasible<FLOWS>(a, t, sm, u0 + v, (int)x0, (int)x1, (int)x3);
      okb |= (k ? 1u : 0u) << (j * VW + v);
      nf += k ? 1 : 0;
      nact += k ? (int)x2 : 0;
      mn0 = min(mn0, k ? x0 : UINT_MAX); mx0 = max(mx0, k ? x0 : 0u);
      mn1 = min(mn1, k ? x1 : UINT_MAX); mx1 = max(mx1, k ? x1 : 0u);
      mn3 = min(mn3, k ? x3 : UINT_MAX); mx3 = max(mx3, k ? x3 : 0u);
      const unsigned y0 = k ? x0 : 0u, y1 = k ? x1 : 0u, y3 = k ? x3 : 0u;
      q0 += (unsigned long long)y0 * y0;
      q1 += (unsigned long long)y1 * y1;
      q3 += (unsigned long long)y3 * y3;
    }
  }
  nf = (int)__reduce_add_sync(NACS_FULL, (unsigned)nf);
  nact = (int)__reduce_add_sync(NACS_FULL, (unsigned)nact);
  mn0 = __reduce_min_sync(NACS_FULL, mn0); mx0 = __reduce_max_sync(NACS_FULL, mx0);
  mn1 = __reduce_min_sync(NACS_FULL, mn1); mx1 = __reduce_max_sync(NACS_FULL, mx1);
  mn3 = __reduce_min_sync(NACS_FULL, mn3); mx3 = __reduce_max_sync(NACS_FULL, mx3);
  v0 = __reduce_max_sync(NACS_FULL, v0); v1 = __reduce_max_sync(NACS_FULL, v1);
  v2 = __reduce_max_sync(NACS_FULL, v2); v3 = __reduce_max_sync(NACS_FULL, v3);
  q0 = warp_sum_u64(q0);
  q1 = warp_sum_u64(q1);
  q3 = warp_sum_u64(q3);
  if (lane == 0) {
    WStats& w = sm.ws[p][warp];
    w.nf = nf; w.nact = nact;
    w.mn[0] = mn0; w.mx[0] = mx0; w.mn[1] = mn1; w.mx[1] = mx1; w.mn[2] = mn3; w.mx[2] = mx3;
    w.vmax[0] = v0; w.vmax[1] = v1; w.vmax[2] = v2; w.vmax[3] = v3;
    w.q[0] = q0; w.q[1] = q1; w.q[2] = q3;
    if (warp == 0) sm.state[p] = b;
  }
  cl.sync();  // this state's statistics and the previous state's keys are visible over DSMEM
  rm_gather(a, t, sm, cl, p, i > 0, p ^ 1);
  __syncthreads();
  if (warp == 0) rm_params(a, t, sm, p);
  if (warp == 1 && i > 0) rm_keys(a, t, sm, p ^ 1);
  __syncthreads();
  if (i > 0) rm_finish<FLOWS>(a, t, sm, cl, p ^ 1);
  TopsisP tp;  // the FP32 fields in registers
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    tp.sf[c] = sm.tp[p].sf[c]; tp.s2p23[c] = sm.tp[p].s2p23[c]; tp.mx[c] = sm.tp[p].mx[c]; tp.mn[c] = sm.tp[p].mn[c];
  }
  tp.p2sq[0] = sm.tp[p].p2sq[0]; tp.p2sq[1] = sm.tp[p].p2sq[1];
  tp.m2sq[0] = sm.tp[p].m2sq[0]; tp.m2sq[1] = sm.tp[p].m2sq[1];
  const bool BAD = sm.BAD[p] != 0;
  const bool live = sm.NF[p] > 0 && !BAD;
  // ----------------------------------------------- a5T: closeness, top-2 keys --
  float s1 = -1.f, s2 = -1.f;  // this thread's best two closeness values (servers i1, i2)
  int i1 = 0, i2 = 0;
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    const int u0 = t.lo + VW * (tid + RM_T * j);
    float sc[VW];
#pragma unroll
    for (int v = 0; v < VW; ++v) {
      const bool k = live && ((okb >> (j * VW + v)) & 1u);
      const float r = topsis32(tp, x[j][0][v], x[j][1][v], x[j][2][v], x[j][3][v]);
      sc[v] = k ? r : 0.f;
      const float rk = k ? r : -1.f;
      const bool g1 = rk > s1, g2 = rk > s2;  // servers ascend: equal scores keep the lower index
      s2 = g1 ? s1 : (g2 ? rk : s2);
      i2 = g1 ? i1 : (g2 ? u0 + v : i2);
      s1 = g1 ? rk : s1;
      i1 = g1 ? u0 + v : i1;
    }
    if (u0 < t.hi) {
      if (a.scores) stv(a.scores + (long long)b * n + u0, sc);
      if (a.mask) {
        const unsigned m = BAD ? 0u : (okb >> (j * VW)) & ((1u << VW) - 1u);
        if (VW == 4) stm(a.mask + (long long)b * n + u0, m);
        else stm2(a.mask + (long long)b * n + u0, m);
      }
    }
  }
  unsigned long long k1 = s1 >= 0.f ? score_key(s1, i1) : 0ull;
  unsigned long long k2 = s2 >= 0.f ? score_key(s2, i2) : 0ull;
  warp_top2(k1, k2);
  if (lane == 0) { sm.wk[p][warp].k1 = k1; sm.wk[p][warp].k2 = k2; }
}

__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_wait(unsigned mb, unsigned parity) {
  asm volatile(
      "{\n .reg .pred P1;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @!P1 bra WAIT_%=;\n}" ::"r"(mb), "r"(parity)
      : "memory");
}

// TMA producer (one thread): the slice's four criteria rows of state b into stage buffer
// `buf` (4 x S int32), completion counted on mbarrier mb
__device__ __forceinline__ void rm_tma(const RankManyArgs& a, const RmThread& t, int b, int* buf, unsigned mb) {
  const int n = a.g.n, S = a.slice;
  const unsigned bytes = 4u * (unsigned)(t.hi - t.lo);  // a multiple of 16 (n, S, stride % 4 == 0)
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(4u * bytes) : "memory");
  const int* sp = a.states + (long long)b * a.stride + t.lo;
#pragma unroll
  for (int c = 0; c < 4; ++c)
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(buf + c * S)),
        "l"(sp + c * n), "r"(bytes), "r"(mb)
        : "memory");
}

// grid = #clusters x C CTAs, cluster dims (C, 1, 1) set at launch.
// TMA: the slices of the cluster's next two states stream into a double-buffered stage in
// shared memory (cp.async.bulk + mbarrier, the async proxy: the cluster barriers of the
// current state do not wait for them); each state's rows go stage -> registers -> stage
// released.  Without 16-byte alignment (n % 4 != 0: k = 2 mod 4) plain loads, no prefetch.
template <int VW, bool TMA, bool FLOWS>
__global__ void __launch_bounds__(RM_T, 1) k_rank_many(RankManyArgs a) {
  extern __shared__ __align__(128) int stage[];  // TMA: [2][4][slice]
  __shared__ RmShared sm;
  __shared__ __align__(8) unsigned long long full[2];
  cg::cluster_group cl = cg::this_cluster();
  RmThread t;
  t.C = (int)cl.num_blocks();
  t.rank = (int)cl.block_rank();
  t.tid = threadIdx.x;
  t.lane = t.tid & 31;
  t.warp = t.tid >> 5;
  t.lo = t.rank * a.slice;
  t.hi = min(a.g.n, t.lo + a.slice);
  t.net = a.path_filter && a.nflow > 0;
  t.e_lo = t.lo < t.hi ? (int)div_h((unsigned)t.lo, a.g.magic_h) : 0;
  t.e_hi = t.lo < t.hi ? (int)div_h((unsigned)(t.hi - 1), a.g.magic_h) : -1;
  const int ncl = gridDim.x / t.C;
  const int cid = blockIdx.x / t.C;
  const int S = a.slice;
  constexpr int NJ = RM_V / VW;
  const bool have = t.lo < t.hi;  // an empty slice (n < C * S) loads nothing
  if (t.tid < 4) sm.cnt[t.tid] = 0ull;
  if (TMA && t.tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&full[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&full[1])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (have) {
      if (cid < a.B) rm_tma(a, t, cid, stage, smem_addr(&full[0]));
      if (cid + ncl < a.B) rm_tma(a, t, cid + ncl, stage + 4 * S, smem_addr(&full[1]));
    }
  }
  __syncthreads();
  int x[NJ][4][VW];
  int i = 0;
  for (int b = cid; b < a.B; b += ncl, ++i) {
    if (TMA) {
      const int sidx = i & 1;
      const int* buf = stage + sidx * 4 * S;
      if (have) mbar_wait(smem_addr(&full[sidx]), (unsigned)((i >> 1) & 1));
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const int o = VW * (t.tid + RM_T * j);
        if (t.lo + o < t.hi) {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int4 v = *reinterpret_cast<const int4*>(buf + c * S + o);
            x[j][c][0] = v.x; x[j][c][1] = v.y; x[j][c][2] = v.z; x[j][c][3] = v.w;
          }
        } else {
#pragma unroll
          for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int v = 0; v < VW; ++v) x[j][c][v] = 0;
        }
      }
      __syncthreads();  // the stage is free: refill it with the state two iterations ahead
      if (t.tid == 0 && have && b + 2 * ncl < a.B) rm_tma(a, t, b + 2 * ncl, stage + sidx * 4 * S, smem_addr(&full[sidx]));
    } else {
      rm_load<VW>(a, t, b, x);
    }
    rm_state<VW, FLOWS>(a, t, sm, cl, b, i, x);
  }
  cl.sync();  // the last state's keys are visible
  if (i > 0) {
    const int q = (i - 1) & 1;
    if (t.warp == 0) {  // warp 0 gathers the last state's keys alone (no statistics pending)
      unsigned long long k1 = 0, k2 = 0;
      for (int r = t.lane; r < t.C * RM_NW; r += 32) {
        const WKeys* w = cl.map_shared_rank(&sm.wk[q][r % RM_NW], r / RM_NW);
        top2_merge(k1, k2, w->k1, w->k2);
      }
      warp_top2(k1, k2);
      if (t.lane == 0) { sm.rk[0].k1 = k1; sm.rk[0].k2 = k2; }
      for (int w = 1 + t.lane; w < RM_NW; w += 32) { sm.rk[w].k1 = 0; sm.rk[w].k2 = 0; }
    }
    __syncthreads();
    if (t.warp == 0) rm_keys(a, t, sm, q);
    __syncthreads();
    rm_finish<FLOWS>(a, t, sm, cl, q);
  }
  if (t.rank == 0 && t.tid == 0 && a.stats && sm.cnt[0]) {
    atomicAdd(&a.stats[ST_POD_STEPS], sm.cnt[0]);
    atomicAdd(&a.stats[ST_FEAS], sm.cnt[1]);
    if (sm.cnt[2]) atomicAdd(&a.stats[ST_FP64], sm.cnt[2]);
    if (sm.cnt[3]) atomicAdd(&a.stats[ST_INVALID], sm.cnt[3]);
  }
  cl.sync();  // no CTA may leave while another still reads its shared memory
}

// Reduce 32 lanes' WStats (exact integers, any order); the result is valid in every lane.
__device__ __forceinline__ void ws_warp_reduce(WStats& x) {
  x.nf = (int)__reduce_add_sync(NACS_FULL, (unsigned)x.nf);
  x.nact = (int)__reduce_add_sync(NACS_FULL, (unsigned)x.nact);
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    x.mn[c] = __reduce_min_sync(NACS_FULL, x.mn[c]);
    x.mx[c] = __reduce_max_sync(NACS_FULL, x.mx[c]);
    x.q[c] = warp_sum_u64(x.q[c]);
  }
#pragma unroll
  for (int c = 0; c < 4; ++c) x.vmax[c] = __reduce_max_sync(NACS_FULL, x.vmax[c]);
}
__device__ __forceinline__ WStats ws_identity() {
  WStats x;
  x.nf = 0; x.nact = 0;
#pragma unroll
  for (int c = 0; c < 3; ++c) { x.mn[c] = UINT_MAX; x.mx[c] = 0; x.q[c] = 0; }
#pragma unroll
  for (int c = 0; c < 4; ++c) x.vmax[c] = 0;
  return x;
}

// =====================================================================================
// Occupancy-2 streaming kernel (16-byte aligned states, no flows/exclusions: the cold
// snapshot stream of §8(d)).  256 threads x 16 servers per CTA (slice of 4096), TWO CTAs of
// different clusters per SM: while one waits at its cluster barrier the other computes.
// A single TMA stage per CTA: the state's rows go stage -> registers, then the next state's
// TMA is issued at once (async proxy: the cluster barrier does not wait for it), so the load
// of state b + #clusters overlaps the whole ranking of state b.
// =====================================================================================
constexpr int RO_V = 16, RO_NJ = RO_V / 4;  // servers per thread; the CTA has T threads (128 or 256)
constexpr int RO_MAXW = 8;

struct RoKey {  // top-2 entry: b = FP32 closeness bits + 1 (0 = none), i = its server, b2 = runner-up bits + 1
  unsigned b1;
  int i1;
  unsigned b2;
};
struct RoShared {
  WStats cs[2];                 // the CTA's statistics of a state (shared-memory atomics of its warps)
  RoKey ks[2][RO_MAXW];         // per-warp top-2 entries
  TopsisP tp[2];
  int NF[2], BAD[2], state[2];
  double argv;
  int argj, best, amb;
  double rd[RO_MAXW];
  int rj[RO_MAXW];
  unsigned long long cnt[4];
  __align__(8) unsigned long long full;
};

__device__ __forceinline__ float sqrt_approx(float x) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
// a5T in FP32 for a FEASIBLE server (mn <= x <= mx, so every difference d is in [0, 2^23)):
// (2^23 + d) as one integer add on the pre-biased bounds, one FMA per scaled difference
// (rounded once), MUFU square roots (<= 2u each) and reciprocal; off F the value is
// meaningless and the caller masks it.  Same error budget as topsis32.
__device__ __forceinline__ float topsis32f(const TopsisP& t, int x0, int x1, int x2, int x3) {
  const float p0 = fmaf(t.sf[0], __int_as_float(t.mxb[0] - x0), -t.s2p23[0]);
  const float m0 = fmaf(t.sf[0], __int_as_float(x0 + t.mnb[0]), -t.s2p23[0]);
  const float p1 = fmaf(t.sf[1], __int_as_float(t.mxb[1] - x1), -t.s2p23[1]);
  const float m1 = fmaf(t.sf[1], __int_as_float(x1 + t.mnb[1]), -t.s2p23[1]);
  const float p3 = fmaf(t.sf[3], __int_as_float(t.mxb[3] - x3), -t.s2p23[3]);
  const float m3 = fmaf(t.sf[3], __int_as_float(x3 + t.mnb[3]), -t.s2p23[3]);
  const float ep2 = fmaf(p3, p3, fmaf(p1, p1, fmaf(p0, p0, x2 ? t.p2sq[1] : t.p2sq[0])));
  const float em2 = fmaf(m3, m3, fmaf(m1, m1, fmaf(m0, m0, x2 ? t.m2sq[1] : t.m2sq[0])));
  const float ep = sqrt_approx(ep2), em = sqrt_approx(em2);
  const float den = __fadd_rn(ep, em);
  return den > 0.f ? __fmul_rn(em, rcp_approx(den)) : 0.f;
}

// Combine top-2 entries (b1, i1, b2) in a warp: the best (largest closeness, then lowest
// server) and the best among everything else (ties with the best count: s1 - s2 = 0).
__device__ __forceinline__ RoKey rokey_warp(RoKey e) {
  const unsigned M = __reduce_max_sync(NACS_FULL, e.b1);
  const int I = (int)__reduce_min_sync(NACS_FULL, e.b1 == M ? (unsigned)e.i1 : 0xFFFFFFFFu);
  const bool win = M != 0 && e.b1 == M && e.i1 == I;
  const unsigned S2 = __reduce_max_sync(NACS_FULL, win ? e.b2 : e.b1);
  RoKey r;
  r.b1 = M;
  r.i1 = I;
  r.b2 = S2;
  return r;
}
__device__ __forceinline__ RoKey rokey_merge(RoKey a, RoKey b) {
  const bool aw = a.b1 > b.b1 || (a.b1 == b.b1 && a.i1 < b.i1);
  RoKey r;
  r.b1 = aw ? a.b1 : b.b1;
  r.i1 = aw ? a.i1 : b.i1;
  r.b2 = aw ? max(a.b2, b.b1) : max(b.b2, a.b1);
  return r;
}

__device__ __forceinline__ void ws_reset(WStats& w) { w = ws_identity(); }

__device__ void ro_params(const RankManyArgs& a, const RmThread& t, RoShared& sm, cg::cluster_group& cl, int p) {
  WStats x = t.lane < t.C ? *cl.map_shared_rank(&sm.cs[p], t.lane) : ws_identity();
  ws_warp_reduce(x);
  const int nf = x.nf, nact = x.nact;
  const int c = t.lane & 3;  // lane c: criterion c's FP64 norm and scale (R12)
  const unsigned long long sq = c == 0 ? x.q[0] : c == 1 ? x.q[1] : c == 2 ? (unsigned long long)nact : x.q[2];
  const double N = sqrt((double)sq);
  const double sdc = N > 0 ? a.wd[c] / N : 0.0;
  double sd[4];
#pragma unroll
  for (int cc = 0; cc < 4; ++cc) sd[cc] = __shfl_sync(NACS_FULL, sdc, cc);
  if (t.lane == 0) {
    TopsisP& tp = sm.tp[p];
    const int mn[4] = {(int)x.mn[0], (int)x.mn[1], nact == nf ? 1 : 0, (int)x.mn[2]};  // f_u in {0,1}
    const int mx[4] = {(int)x.mx[0], (int)x.mx[1], nact > 0 ? 1 : 0, (int)x.mx[2]};
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
      tp.mn[cc] = mn[cc];
      tp.mx[cc] = mx[cc];
      tp.sd[cc] = sd[cc];
      tp.sf[cc] = (float)sd[cc];
      tp.s2p23[cc] = (float)sd[cc] * 8388608.0f;
      tp.mxb[cc] = 0x4B000000 + mx[cc];
      tp.mnb[cc] = 0x4B000000 - mn[cc];
    }
    const float q2 = __fmul_rn(tp.sf[2], tp.sf[2]);
    tp.p2sq[0] = mx[2] - 0 ? q2 : 0.f;
    tp.p2sq[1] = mx[2] - 1 ? q2 : 0.f;
    tp.m2sq[0] = 0 - mn[2] ? q2 : 0.f;
    tp.m2sq[1] = 1 - mn[2] ? q2 : 0.f;
    sm.NF[p] = nf;
    // R5: every value an exact FP32 integer in range (device-pointer states validated here)
    sm.BAD[p] = x.vmax[0] > (unsigned)a.g.cpu_cap || x.vmax[1] > (unsigned)a.g.ram_cap || x.vmax[2] > 1u ||
                x.vmax[3] > (unsigned)a.g.link_cap;
  }
}

// top-2 of slot q's state from the C x 8 warp entries; ambiguity (gap <= 2^-17)
template <int NW>
__device__ void ro_keys(const RankManyArgs& a, const RmThread& t, RoShared& sm, cg::cluster_group& cl, int q) {
  RoKey e;
  e.b1 = 0; e.i1 = 0x7FFFFFFF; e.b2 = 0;
  for (int j = t.lane; j < t.C * NW; j += 32) e = rokey_merge(e, *cl.map_shared_rank(&sm.ks[q][j % NW], j / NW));
  e = rokey_warp(e);
  if (t.lane == 0) {
    const float s1 = __uint_as_float(e.b1 - 1u), s2 = __uint_as_float(e.b2 - 1u);
    const bool live = sm.NF[q] > 0 && !sm.BAD[q];
    sm.best = e.b1 ? e.i1 : -1;
    sm.amb = live && e.b1 && (a.exact64 || (e.b2 != 0u && s1 - s2 <= kTopsisDelta));
    sm.argv = (double)s1;
  }
}

// Finish slot q's state after ro_keys: FP64 re-decision when ambiguous (the state's slice is
// read again; two more cluster barriers; every CTA takes the branch), then rank 0 writes.
template <int T>
__device__ void ro_finish(const RankManyArgs& a, const RmThread& t, RoShared& sm, cg::cluster_group& cl, int q) {
  constexpr int NW = T / 32;
  const bool amb = sm.amb;
  const int b = sm.state[q];
  if (amb) {
    const float thr = a.exact64 ? -1.0f : (float)sm.argv - 2.0f * kTopsisDelta;
    const TopsisP& tp = sm.tp[q];
    const int n = a.g.n;
    const int* st = a.states + (long long)b * a.stride;
    double bv = -DBL_MAX;
    int bj = -1;
    for (int u = t.lo + t.tid; u < t.hi; u += T) {
      const int x0 = st[u], x1 = st[n + u], x2 = st[2 * n + u], x3 = st[3 * n + u];
      if (!(x0 >= a.dc && x1 >= a.dr)) continue;
      if (topsis32f(tp, x0, x1, x2, x3) < thr) continue;
      const double r = topsis64(tp, x0, x1, x2, x3);
      if (r > bv || (r == bv && u < bj)) { bv = r; bj = u; }
    }
    warp_argmax64(bv, bj);
    __syncthreads();  // everyone has read argv (thr) before it is rewritten
    if (t.lane == 0) { sm.rd[t.warp] = bv; sm.rj[t.warp] = bj; }
    __syncthreads();
    if (t.warp == 0) {
      bv = t.lane < NW ? sm.rd[t.lane] : -DBL_MAX;
      bj = t.lane < NW ? sm.rj[t.lane] : -1;
      warp_argmax64(bv, bj);
      if (t.lane == 0) { sm.argv = bv; sm.argj = bj; }
    }
    cl.sync();  // every CTA's FP64 candidate is visible
    if (t.warp == 0) {
      bv = -DBL_MAX;
      bj = -1;
      if (t.lane < t.C) {
        const double* v = cl.map_shared_rank(&sm.argv, t.lane);
        const int* j = cl.map_shared_rank(&sm.argj, t.lane);
        if (*j >= 0) { bv = *v; bj = *j; }
      }
      warp_argmax64(bv, bj);
      if (t.lane == 0) sm.best = bj;
    }
    cl.sync();  // nobody rewrites argv / argj before every CTA has read them
  }
  if (t.rank == 0 && t.tid == 0) {
    const int NF = sm.NF[q], BAD = sm.BAD[q];
    a.best[b] = BAD ? -2 : (NF > 0 ? sm.best : -1);
    sm.cnt[0] += 1;
    sm.cnt[1] += (unsigned long long)NF;
    sm.cnt[2] += amb ? 1 : 0;
    sm.cnt[3] += BAD ? 1 : 0;
  }
}

// TMA store (async proxy) of a CTA's score row: shared -> global, one bulk group
__device__ __forceinline__ void ro_store_scores(const float* src, float* dst, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_addr(src)),
               "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

template <int T>
__global__ void __launch_bounds__(T, 512 / T) k_rank_occ(RankManyArgs a) {
  constexpr int RO_T = T;
  extern __shared__ __align__(128) int stage[];  // [4][slice] rows | [2][slice] scores
  __shared__ RoShared sm;
  cg::cluster_group cl = cg::this_cluster();
  RmThread t;
  t.C = (int)cl.num_blocks();
  t.rank = (int)cl.block_rank();
  t.tid = threadIdx.x;
  t.lane = t.tid & 31;
  t.warp = t.tid >> 5;
  t.lo = t.rank * a.slice;
  t.hi = min(a.g.n, t.lo + a.slice);
  t.net = false;
  t.e_lo = 0;
  t.e_hi = -1;
  const int ncl = gridDim.x / t.C;
  const int cid = blockIdx.x / t.C;
  const int S = a.slice, n = a.g.n;
  const bool have = t.lo < t.hi;
  float* scbuf = reinterpret_cast<float*>(stage + 4 * S);  // [2][S]
  const unsigned mb = smem_addr(&sm.full);
  if (t.tid < 4) sm.cnt[t.tid] = 0ull;
  if (t.tid == 0) {
    ws_reset(sm.cs[0]);
    ws_reset(sm.cs[1]);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (have && cid < a.B) rm_tma(a, t, cid, stage, mb);
  }
  __syncthreads();
  int i = 0, prev_b = -1;
  for (int b = cid; b < a.B; b += ncl, ++i) {
    const int p = i & 1;
    // ------------------------------------------------ a0: stage -> registers --
    int x[RO_NJ][4][4];
    if (have) mbar_wait(mb, (unsigned)(i & 1));
#pragma unroll
    for (int j = 0; j < RO_NJ; ++j) {
      const int o = 4 * (t.tid + RO_T * j);
      if (t.lo + o < t.hi) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int4 v = *reinterpret_cast<const int4*>(stage + c * S + o);
          x[j][c][0] = v.x; x[j][c][1] = v.y; x[j][c][2] = v.z; x[j][c][3] = v.w;
        }
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int v = 0; v < 4; ++v) x[j][c][v] = 0;
      }
    }
    __syncthreads();  // the stage is free (and the previous state's scores are in scbuf)
    if (t.tid == 0 && have) {
      if (b + ncl < a.B) rm_tma(a, t, b + ncl, stage, mb);  // the next state streams in during this one
      if (a.scores && prev_b >= 0) {
        ro_store_scores(scbuf + (p ^ 1) * S, a.scores + (long long)prev_b * n + t.lo, 4u * (unsigned)(t.hi - t.lo));
        // the score buffer of this state (written below) was stored two states ago: done reading?
        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      }
    }
    // --------------------------------------------------- a3 + a4: filter, stats --
    unsigned okb = 0;
    WStats w = ws_identity();
#pragma unroll
    for (int j = 0; j < RO_NJ; ++j)
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const unsigned x0 = (unsigned)x[j][0][v], x1 = (unsigned)x[j][1][v], x2 = (unsigned)x[j][2][v],
                       x3 = (unsigned)x[j][3][v];
        w.vmax[0] = max(w.vmax[0], x0); w.vmax[1] = max(w.vmax[1], x1);
        w.vmax[2] = max(w.vmax[2], x2); w.vmax[3] = max(w.vmax[3], x3);
        if ((int)x0 >= a.dc && (int)x1 >= a.dr) {  // demands > 0: padding (values 0) never passes
          okb |= 1u << (j * 4 + v);
          w.nf += 1;
          w.nact += (int)x2;
          w.mn[0] = min(w.mn[0], x0); w.mx[0] = max(w.mx[0], x0);
          w.mn[1] = min(w.mn[1], x1); w.mx[1] = max(w.mx[1], x1);
          w.mn[2] = min(w.mn[2], x3); w.mx[2] = max(w.mx[2], x3);
          w.q[0] += (unsigned long long)x0 * x0;
          w.q[1] += (unsigned long long)x1 * x1;
          w.q[2] += (unsigned long long)x3 * x3;
        }
      }
    {  // into the CTA slot: 32-bit warp reductions + one lane's atomics; 64-bit sums by atomics
      WStats& cs = sm.cs[p];
      // a thread's sums are < 16 x 2^46 = 2^50: two 25-bit halves sum exactly in 32 bits over
      // a warp (32 x 2^25 = 2^30), so each 64-bit sum is two redux.sync
      unsigned long long qw[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const unsigned lo = __reduce_add_sync(NACS_FULL, (unsigned)(w.q[c] & 0x1FFFFFFull));
        const unsigned hi = __reduce_add_sync(NACS_FULL, (unsigned)(w.q[c] >> 25));
        qw[c] = ((unsigned long long)hi << 25) + lo;
      }
      const int nf = (int)__reduce_add_sync(NACS_FULL, (unsigned)w.nf);
      const int nact = (int)__reduce_add_sync(NACS_FULL, (unsigned)w.nact);
      unsigned mn[3], mx[3], vm[4];
#pragma unroll
      for (int c = 0; c < 3; ++c) { mn[c] = __reduce_min_sync(NACS_FULL, w.mn[c]); mx[c] = __reduce_max_sync(NACS_FULL, w.mx[c]); }
#pragma unroll
      for (int c = 0; c < 4; ++c) vm[c] = __reduce_max_sync(NACS_FULL, w.vmax[c]);
      if (t.lane == 0) {
#pragma unroll
        for (int c = 0; c < 3; ++c) atomicAdd(&cs.q[c], qw[c]);
        atomicAdd(&cs.nf, nf);
        atomicAdd(&cs.nact, nact);
#pragma unroll
        for (int c = 0; c < 3; ++c) { atomicMin(&cs.mn[c], mn[c]); atomicMax(&cs.mx[c], mx[c]); }
#pragma unroll
        for (int c = 0; c < 4; ++c) atomicMax(&cs.vmax[c], vm[c]);
        if (t.warp == 0) sm.state[p] = b;
      }
    }
    cl.sync();  // this state's statistics and the previous state's keys are visible over DSMEM
    if (t.warp == 0) ro_params(a, t, sm, cl, p);
    if (t.warp == 1 && i > 0) ro_keys<T / 32>(a, t, sm, cl, p ^ 1);
    __syncthreads();
    if (t.tid == 0) ws_reset(sm.cs[p ^ 1]);  // every CTA has read the previous state's slot
    if (i > 0) ro_finish<T>(a, t, sm, cl, p ^ 1);
    // ----------------------------------------------- a5T: closeness, top-2 keys --
    TopsisP tp;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      tp.sf[c] = sm.tp[p].sf[c]; tp.s2p23[c] = sm.tp[p].s2p23[c]; tp.mxb[c] = sm.tp[p].mxb[c]; tp.mnb[c] = sm.tp[p].mnb[c];
    }
    tp.p2sq[0] = sm.tp[p].p2sq[0]; tp.p2sq[1] = sm.tp[p].p2sq[1];
    tp.m2sq[0] = sm.tp[p].m2sq[0]; tp.m2sq[1] = sm.tp[p].m2sq[1];
    if (sm.BAD[p] || sm.NF[p] == 0) okb = 0;
    float s1 = -1.f, s2 = -1.f;
    int i1 = 0;
#pragma unroll
    for (int j = 0; j < RO_NJ; ++j) {
      const int o = 4 * (t.tid + RO_T * j);
      const int u0 = t.lo + o;
      float sc[4];
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const bool k = (okb >> (j * 4 + v)) & 1u;
        const float r = topsis32f(tp, x[j][0][v], x[j][1][v], x[j][2][v], x[j][3][v]);
        sc[v] = k ? r : 0.f;
        const float rk = k ? r : -1.f;
        const bool g1 = rk > s1;  // servers ascend: equal scores keep the lower index
        s2 = g1 ? s1 : fmaxf(s2, rk);
        i1 = g1 ? u0 + v : i1;
        s1 = g1 ? rk : s1;
      }
      if (u0 < t.hi) {
        if (a.scores) *reinterpret_cast<float4*>(scbuf + p * S + o) = make_float4(sc[0], sc[1], sc[2], sc[3]);
        if (a.mask) stm(a.mask + (long long)b * n + u0, (okb >> (j * 4)) & 15u);
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // scores -> the async proxy (TMA store)
    RoKey e;
    e.b1 = s1 >= 0.f ? __float_as_uint(s1) + 1u : 0u;
    e.i1 = i1;
    e.b2 = s2 >= 0.f ? __float_as_uint(s2) + 1u : 0u;
    e = rokey_warp(e);
    if (t.lane == 0) sm.ks[p][t.warp] = e;
    prev_b = b;
  }
  cl.sync();  // the last state's keys are visible
  if (i > 0) {
    const int q = (i - 1) & 1;
    if (t.warp == 0) ro_keys<T / 32>(a, t, sm, cl, q);
    __syncthreads();
    ro_finish<T>(a, t, sm, cl, q);
    if (t.tid == 0 && have && a.scores) {
      ro_store_scores(scbuf + q * S, a.scores + (long long)prev_b * n + t.lo, 4u * (unsigned)(t.hi - t.lo));
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
  }
  if (t.rank == 0 && t.tid == 0 && a.stats && sm.cnt[0]) {
    atomicAdd(&a.stats[ST_POD_STEPS], sm.cnt[0]);
    atomicAdd(&a.stats[ST_FEAS], sm.cnt[1]);
    if (sm.cnt[2]) atomicAdd(&a.stats[ST_FP64], sm.cnt[2]);
    if (sm.cnt[3]) atomicAdd(&a.stats[ST_INVALID], sm.cnt[3]);
  }
  cl.sync();  // no CTA may leave while another still reads its shared memory
}

// ------------------------------------------------------------------ host ---
int rank_many_cluster(const Geo& g) { return (g.n + RM_S - 1) / RM_S; }

cudaError_t launch_rank_many(const RankManyArgs& a0, int num_sms, cudaStream_t st) {
  RankManyArgs a = a0;
  if (rank_many_cluster(a.g) > 16) return cudaErrorInvalidValue;
  const bool v4 = (a.g.n % 4 == 0) && (a.stride % 4 == 0) && ((uintptr_t)a.states % 16 == 0);
  const bool flows = a.nflow > 0 || a.nex > 0;
  const char* kenv = getenv("NACS_RANK_KERNEL");  // experiment knob: "many" | "occ256"
  // (k_rank_occ stores the scores with TMA bulk copies: 16-byte aligned rows)
  const bool occ = v4 && !flows && ((uintptr_t)a.scores % 16 == 0) && !(kenv && !strcmp(kenv, "many"));
  // k_rank_occ: 128-thread CTAs (4 per SM) when one CTA holds the whole state (n <= 2048: no
  // cluster barrier at all), else 256 (4096-server slices, 2 per SM: at k=32, 4 CTAs of 2048
  // measured 3.47 TB/s against 4.20); k_rank_many: 512 threads, 4096-server slices
  const bool occ128 = occ && a.g.n <= 2048 && !(kenv && !strcmp(kenv, "occ256"));
  const int T = occ ? (occ128 ? 128 : 256) : RM_T;
  const int per_cta = occ ? T * RO_V : RM_S;
  const int C = (a.g.n + per_cta - 1) / per_cta;
  const int VW = v4 ? 4 : 2;
  // slices of <= per_cta servers, a multiple of VW so that vector accesses stay aligned
  int S = (a.g.n + C - 1) / C;
  S = (S + VW - 1) / VW * VW;
  a.slice = S;
  void (*kern)(RankManyArgs) = occ ? (occ128 ? k_rank_occ<128> : k_rank_occ<256>)
                               : v4 ? (flows ? k_rank_many<4, true, true> : k_rank_many<4, true, false>)
                                    : (flows ? k_rank_many<2, false, true> : k_rank_many<2, false, false>);
  // dynamic shared memory: occ = the row stage + 2 score rows (6 S int32); many = 2 row stages
  const size_t dyn = occ ? 6 * sizeof(int) * (size_t)S : v4 ? 2 * 4 * sizeof(int) * (size_t)S : 0;
  const int kid = occ ? (occ128 ? 3 : 2) : flows;
  static int max_clusters[2][4][17] = {};
  static bool dyn_set[4] = {};
  int& mc = max_clusters[v4][kid][C];
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(T, 1, 1);
  cfg.dynamicSmemBytes = dyn;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e;
  if (v4 && !dyn_set[kid]) {  // the variant's largest dynamic shared memory
    const int maxdyn = occ ? 6 * 4 * T * RO_V : 8 * 4 * RM_S;
    if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, maxdyn)) != cudaSuccess) return e;
    dyn_set[kid] = true;
  }
  if (mc == 0) {
    if (C > 8 && (e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)) != cudaSuccess)
      return e;
    cfg.gridDim = dim3(C * num_sms, 1, 1);
    if ((e = cudaOccupancyMaxActiveClusters(&mc, kern, &cfg)) != cudaSuccess) return e;
    if (mc <= 0) return cudaErrorInvalidConfiguration;
  }
  const int ncl = a.B < mc ? a.B : mc;
  if (ncl <= 0) return cudaSuccess;
  cfg.gridDim = dim3(C * ncl, 1, 1);
  return cudaLaunchKernelEx(&cfg, kern, a);
}

}  // namespace nacs
