// nacs_kernels.cu — sm_100a kernels of libnacs: one pod step = feasibility filter,
// per-criterion statistics, AHP or TOPSIS scoring, argmax, commit (§V,
// P:298-386; readings R1-R24 in DESIGN.md).
//
// Execution model.  A CTA runs whole requests: for every pod (ascending id, R15) it
// builds the pod's flows to placed peers (a1-a2), marks fabric-infeasible edge switches
// (a2), filters servers and reduces the criteria statistics (a3-a4), scores the feasible
// servers and reduces a top-2 argmax key (a5-a7), then one warp commits (a8).  The
// request end tops allocations up (a9).
//   * k_batch: persistent CTAs; each holds a private copy of the whole snapshot in
//     shared memory (loaded once per CTA with a TMA bulk copy) and mutates it in place;
//     an undo log restores it after every request (R21 snapshot isolation).
//   * k_sequential: one CTA, requests in order, in place on the global state (the
//     paper's online semantics); a rejected request is rolled back (R20).
//   * k_rank: one CTA, one pod query, no commit.
//
// Numerics.  All state is integer.  Criteria are read as int32 and every difference
// (x - min, max - x) is taken in integers, then converted exactly to FP32 with the
// 2^23 magic-number trick (no I2F on the hot loop).  TOPSIS norms are exact integer sums
// of squares (64-bit).  Scores are FP32; an argmax whose top-2 FP32 gap is inside the
// derived FP32 error bound is re-decided in FP64 over the near-max candidates (R14).
#include <cooperative_groups.h>

#include <cfloat>
#include <cstdio>
#include <cstdlib>
#include <climits>
#include <cstdint>

#include "nacs_device.cuh"

// Debug builds (-DNACS_CHECKS): bounds checks of the cluster engines' index arithmetic trap
// with a message (python paper_1909_07673_b200/build.py exp_checks.so -DNACS_CHECKS, then
// NACS_LIB=... on the GPU tests).
#ifdef NACS_CHECKS
#define NACS_DCHECK(cond)                                                                   \
  do {                                                                                     \
    if (!(cond)) {                                                                         \
      printf("NACS_CHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__, \
             (int)blockIdx.x, (int)threadIdx.x);                                           \
      __trap();                                                                            \
    }                                                                                      \
  } while (0)
#else
#define NACS_DCHECK(cond) \
  do {                    \
  } while (0)
#endif

namespace nacs {

#define FULL 0xffffffffu

// ---------------------------------------------------------------- helpers ----
__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
// AHP: relative error of PG in FP32 <= (96 + 2*ceil(nf/32)) u; ambiguous if the
// relative top-2 gap is <= 2 x that.
// (u = 2^-24; reciprocal sums in FP32 chunks of <= 32 terms accumulated in FP64, linear
// parts from exact prefix sums: PG relative error <= 82u, independent of nf)
__device__ __forceinline__ float ahp_delta_rel(int nf) {
  (void)nf;
  return 2.0f * 96.0f * 5.9604644775390625e-08f;
}

// ------------------------------------------------------------ scratch -------
struct Scratch {
  // request
  int nC, nV, P, req_ok;
  int cpod[MAXC];
  int pod_cpu[MAXC], pod_ram[MAXC], pod_srv[MAXC];
  int vpath[MAXV];
  // pod step
  int p, dc, dr, nflow, sumD, G, vm;
  int fv[MAXF], fD[MAXF], fok[MAXF], fpath[MAXF], fexcl[MAXF];
  unsigned pm[MAXK];
  int fail, log_n, log_mark;
  // a lower bound of every fabric (edge-agg, agg-core) residual of the state (0 = unknown):
  // a flow with D <= minfab passes every edge switch, so its fabric tables are skipped (exact)
  int minfab, minfab0;
  // statistics over the feasible set F
  int nf, nact, mn[4], mx[4];
  unsigned long long sq[4];
  float sf[4], s2p23[4];
  double sd[4];
  // AHP per-criterion configuration
  int ahp_const[4];
  float ahp_scale[4];
  double ahp_scaled[4];
  float L1[4];
  double L1d[4];
  // selection
  unsigned long long key1, key2;
  int best, amb;
  float thr;
  double bestv;
  // block reductions
  int red_i[MAXW][8];
  unsigned long long red_u[MAXW][3];
  unsigned long long red_k[MAXW][2];
  double red_d[MAXW];
  int red_j[MAXW];
  int scan[MAXW];
  double scand[MAXW][2];
  double scand_total[2];
  int scan_total;
  int lvK, m1, nd, ntouched, touch_over, presorted;
  // cluster-wide scans (k_sh_levels): this CTA's totals, read by the others over DSMEM
  // (double-buffered by call parity), and the scan's result
  int cl_pub[2];
  double cl_pubd[2][2];
  int cl_base, cl_total;
  double cl_based[2], cl_totald[2];
  int touched[2 * MAXC];   // servers with changed criteria in the current request (AHP)
  float dval[2 * MAXC];    // dirty feasible values / servers of a pod step, sorted
  int dsrv[2 * MAXC];
  // request fetch (batch)
  int next_req;
  // counters (thread 0)
  unsigned long long c_steps, c_retries, c_fp64, c_invalid, c_feas, c_pairs;
};

struct Ctx {
  Geo g;
  Opt o;
  int* st;             // state words (shared memory in k_batch, global otherwise)
  const int* cr;       // criteria rows cpu | ram | act | bandwidth criterion (= st, or the
                       // logical-bandwidth table of nacs_rank_* with bw_criterion = 1)
  const int* snap;     // global snapshot (k_batch) for reference
  Scratch* s;
  unsigned* maskw;     // [nW] feasibility bitmap of the current pod step
  unsigned* f0w;       // [nW] R25: the feasible set of the request's first pod step
  unsigned* special;   // [nW] flow servers and excluded servers of the pod step
  unsigned* edgebad;   // [nEW] edge switches some flow cannot reach with its demand
  unsigned* spok = nullptr;  // k_seq_cluster: [nW] the special servers' own verdict (a flow
                             // server not excluded and, with path_filter, fok), so the filter
                             // needs no per-server flow search
  // AHP workspace (ahp_carve): presorted orders, sorted levels, prefix sums
  unsigned short* perm;  // [3][n2] servers in ascending CPU, RAM, access-bandwidth order
  unsigned* dirty;       // [nW] servers whose criteria the current request has changed
  float* pg;             // [n] FP32 global priorities, by server
  int* lvl;              // [n] level (rank of distinct value) of each server, current criterion
  float* keys;           // [n2] sorted feasible values
  int* sidx;             // [n2] their servers
  float* keys2;          // [n2] merge buffer
  int* sidx2;            // [n2]
  int* lst;            // [n2+1] first sorted position of each level
  float2* lvm;         // [n2] (value, multiplicity) per level
  float2* lvw;         // [n2] (value, multiplicity / column sum) per level
  double* pa;          // [n2+2] exclusive prefix sums (multiplicity-weighted)
  double* pb;          // [n2+2] exclusive prefix sums (multiplicity-weighted values)
  float* l2;           // [n2] L2 per level
  double* w64;         // FP64 re-decision: [n2] per-level weights + [nfcap] priorities (global)
  int nfcap;
  int2* ulog;          // undo log (global)
  int* const* mirr = nullptr;  // k_seq_cluster: every CTA's shared-memory copy of its share of the
                              // per-server rows (cluster addresses), kept current by st_set
  int tid, B, NW, lane, warp;
  int nW, nEW;
};

#ifdef NACS_SEQC_PROF  // experiment builds: per-phase time of the leader CTA (device printf at the end)
__shared__ unsigned long long seqc_prof_[24], seqc_last_;
#ifdef NACS_SEQC_CYCLES  // SM cycles instead of nanoseconds
#define SEQC_CLOCK() ((unsigned long long)clock64())
#else
__device__ __forceinline__ unsigned long long seqc_gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define SEQC_CLOCK() seqc_gt()
#endif
#define SEQC_T(i)                                                                  \
  do {                                                                             \
    if (blockIdx.x == 0 && threadIdx.x == 0) {                                     \
      unsigned long long now_;                                                     \
      now_ = SEQC_CLOCK();                                                         \
      seqc_prof_[i] += now_ - seqc_last_;                                          \
      seqc_last_ = now_;                                                           \
    }                                                                              \
  } while (0)
#else
#define SEQC_T(i) \
  do {            \
  } while (0)
#endif

// ------------------------------------------------------- undo log (1 thread) --
// k_seq_cluster's row copies: server u of criterion row q lives in CTA (u / 1024) mod C at
// q * SQC_M + (u / (SQC_T C)) * SQC_T + u mod SQC_T (its grid-stride share, see seqc_filter)
#ifndef NACS_SEQC_T
#define NACS_SEQC_T 512
#endif
constexpr int SQC_T = NACS_SEQC_T;  // threads per CTA (a power of two)
constexpr int SQC_M = 4096;         // servers per CTA: C = 16 covers k = 64
constexpr int SQ_J = SQC_M / SQC_T; // servers per thread, kept in registers over a pod step
// (C, the cluster size, is a power of two: seq_cluster_size)
__device__ __forceinline__ int* mirror_ptr(const Ctx& c, int off) {
  const int n = c.g.n;
  const int q = (off >= n) + (off >= 2 * n) + (off >= 3 * n);
  const int u = off - q * n;
  const int C = (int)gridDim.x;
  NACS_DCHECK(off >= 0 && q < 4 && u >= 0 && u < n && (C & (C - 1)) == 0 && (u >> (__ffs(C * SQC_T) - 1)) < SQ_J);
  return c.mirr[(u / SQC_T) & (C - 1)] + q * SQC_M + ((u >> (__ffs(C * SQC_T) - 1)) * SQC_T) + (u & (SQC_T - 1));
}
__device__ __forceinline__ void mirror_put(const Ctx& c, int off, int val) { *mirror_ptr(c, off) = val; }
// A state word for the thread-0 chains: a per-server row word from the cluster copy (a
// distributed-shared-memory round trip instead of an L2 one), else the global state.
__device__ __forceinline__ int st_get(const Ctx& c, int off) {
  return c.mirr && off < 4 * c.g.n ? *mirror_ptr(c, off) : c.st[off];
}
__device__ __forceinline__ void st_set(Ctx& c, int off, int val) {
  Scratch* s = c.s;
  c.ulog[s->log_n] = make_int2(off, st_get(c, off));
  s->log_n += 1;
  c.st[off] = val;
  if (c.mirr && off < 4 * c.g.n) mirror_put(c, off, val);
  if (off >= 4 * c.g.n && val < s->minfab) s->minfab = val;  // commits only lower the bound
  if (c.dirty && off < 4 * c.g.n) {  // AHP: the server leaves its presorted position
    const int u = off % c.g.n;
    if (!((c.dirty[u >> 5] >> (u & 31)) & 1u)) {
      c.dirty[u >> 5] |= 1u << (u & 31);
      if (s->ntouched < 2 * MAXC) s->touched[s->ntouched] = u;
      else s->touch_over = 1;
      s->ntouched += 1;
    }
  }
}
// st_set with the word's current value already known (no reload: on global state a reload
// after the previous store costs a full L2 round trip in the thread-0 commit chain)
__device__ __forceinline__ void st_set_v(Ctx& c, int off, int old, int val) {
  Scratch* s = c.s;
  c.ulog[s->log_n] = make_int2(off, old);
  s->log_n += 1;
  c.st[off] = val;
  if (c.mirr && off < 4 * c.g.n) mirror_put(c, off, val);
  if (off >= 4 * c.g.n && val < s->minfab) s->minfab = val;
  if (c.dirty && off < 4 * c.g.n) {  // AHP: the server leaves its presorted position (as st_set)
    const int u = off % c.g.n;
    if (!((c.dirty[u >> 5] >> (u & 31)) & 1u)) {
      c.dirty[u >> 5] |= 1u << (u & 31);
      if (s->ntouched < 2 * MAXC) s->touched[s->ntouched] = u;
      else s->touch_over = 1;
      s->ntouched += 1;
    }
  }
}
__device__ __forceinline__ void undo_to(Ctx& c, int mark) {
  Scratch* s = c.s;
  for (int i = s->log_n - 1; i >= mark; --i) {
    int2 e = c.ulog[i];
    c.st[e.x] = e.y;
    if (c.mirr && e.x < 4 * c.g.n) mirror_put(c, e.x, e.y);
  }
  s->log_n = mark;
}

// ------------------------------------------------------------ reductions -----
// Block-wide top-2 of 64-bit keys; result in s->key1, s->key2.  All threads call.
__device__ void block_top2(Ctx& c, unsigned long long k1, unsigned long long k2) {
  Scratch* s = c.s;
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long b1 = __shfl_xor_sync(FULL, k1, o);
    unsigned long long b2 = __shfl_xor_sync(FULL, k2, o);
    top2_merge(k1, k2, b1, b2);
  }
  if (c.lane == 0) { s->red_k[c.warp][0] = k1; s->red_k[c.warp][1] = k2; }
  __syncthreads();
  if (c.warp == 0) {
    k1 = c.lane < c.NW ? s->red_k[c.lane][0] : 0ull;
    k2 = c.lane < c.NW ? s->red_k[c.lane][1] : 0ull;
    for (int o = 16; o > 0; o >>= 1) {
      unsigned long long b1 = __shfl_xor_sync(FULL, k1, o);
      unsigned long long b2 = __shfl_xor_sync(FULL, k2, o);
      top2_merge(k1, k2, b1, b2);
    }
    if (c.lane == 0) { s->key1 = k1; s->key2 = k2; }
  }
  __syncthreads();
}

// Block-wide argmax of (double value, index): larger value, then lower index.
__device__ void block_argmax64(Ctx& c, double v, int j) {
  Scratch* s = c.s;
  for (int o = 16; o > 0; o >>= 1) {
    double bv = __shfl_xor_sync(FULL, v, o);
    int bj = __shfl_xor_sync(FULL, j, o);
    if (bv > v || (bv == v && (unsigned)bj < (unsigned)j)) { v = bv; j = bj; }
  }
  if (c.lane == 0) { s->red_d[c.warp] = v; s->red_j[c.warp] = j; }
  __syncthreads();
  if (c.warp == 0) {
    v = c.lane < c.NW ? s->red_d[c.lane] : -DBL_MAX;
    j = c.lane < c.NW ? s->red_j[c.lane] : -1;
    for (int o = 16; o > 0; o >>= 1) {
      double bv = __shfl_xor_sync(FULL, v, o);
      int bj = __shfl_xor_sync(FULL, j, o);
      if (bv > v || (bv == v && (unsigned)bj < (unsigned)j)) { v = bv; j = bj; }
    }
    if (c.lane == 0) { s->best = j; s->bestv = v; }
  }
  __syncthreads();
}

// Exclusive block scan of one int per thread.
__device__ int block_exscan(Ctx& c, int x) {
  Scratch* s = c.s;
  int inc = x;
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(FULL, inc, o);
    if (c.lane >= o) inc += y;
  }
  if (c.lane == 31) s->scan[c.warp] = inc;
  __syncthreads();
  if (c.warp == 0) {
    int t = c.lane < c.NW ? s->scan[c.lane] : 0;
    int ti = t;
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(FULL, ti, o);
      if (c.lane >= o) ti += y;
    }
    if (c.lane < c.NW) s->scan[c.lane] = ti - t;
  }
  __syncthreads();
  int r = s->scan[c.warp] + inc - x;
  __syncthreads();
  return r;
}

// Exclusive block scan of two doubles per thread (returned in place).
__device__ void block_exscan_d2(Ctx& c, double& a, double& b) {
  Scratch* s = c.s;
  double ia = a, ib = b;
  for (int o = 1; o < 32; o <<= 1) {
    double ya = __shfl_up_sync(FULL, ia, o), yb = __shfl_up_sync(FULL, ib, o);
    if (c.lane >= o) { ia += ya; ib += yb; }
  }
  if (c.lane == 31) { s->scand[c.warp][0] = ia; s->scand[c.warp][1] = ib; }
  __syncthreads();
  if (c.warp == 0) {
    double ta = c.lane < c.NW ? s->scand[c.lane][0] : 0.0, tb = c.lane < c.NW ? s->scand[c.lane][1] : 0.0;
    double xa = ta, xb = tb;
    for (int o = 1; o < 32; o <<= 1) {
      double ya = __shfl_up_sync(FULL, xa, o), yb = __shfl_up_sync(FULL, xb, o);
      if (c.lane >= o) { xa += ya; xb += yb; }
    }
    if (c.lane < c.NW) { s->scand[c.lane][0] = xa - ta; s->scand[c.lane][1] = xb - tb; }
  }
  __syncthreads();
  const double ra = s->scand[c.warp][0] + ia - a, rb = s->scand[c.warp][1] + ib - b;
  __syncthreads();
  a = ra;
  b = rb;
}

// Warp segments for coalesced, stable block-wide scans: warp w owns a contiguous range
// [s0, s1) of [0, N), 32 elements per step; positions inside a step come from ballots.
__device__ __forceinline__ void warp_seg(const Ctx& c, int N, int& s0, int& s1) {
  const int seg = ((N + c.NW - 1) / c.NW + 31) & ~31;
  s0 = min(c.warp * seg, N);
  s1 = min(s0 + seg, N);
}
// Exclusive scan over the warps of one int per warp; *total = the sum.  All threads.
__device__ int warp_exscan(Ctx& c, int x, int* total) {
  Scratch* s = c.s;
  if (c.lane == 0) s->scan[c.warp] = x;
  __syncthreads();
  if (c.warp == 0) {
    const int t = c.lane < c.NW ? s->scan[c.lane] : 0;
    int ti = t;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(FULL, ti, o);
      if (c.lane >= o) ti += y;
    }
    if (c.lane < c.NW) s->scan[c.lane] = ti - t;
    if (c.lane == 31) s->scan_total = ti;
  }
  __syncthreads();
  const int r = s->scan[c.warp];
  *total = s->scan_total;
  __syncthreads();
  return r;
}
// Same for two doubles per warp.
__device__ void warp_exscan_d2(Ctx& c, double& a, double& b, double* ta, double* tb) {
  Scratch* s = c.s;
  if (c.lane == 0) { s->scand[c.warp][0] = a; s->scand[c.warp][1] = b; }
  __syncthreads();
  if (c.warp == 0) {
    const double xa = c.lane < c.NW ? s->scand[c.lane][0] : 0.0, xb = c.lane < c.NW ? s->scand[c.lane][1] : 0.0;
    double ia = xa, ib = xb;
    for (int o = 1; o < 32; o <<= 1) {
      const double ya = __shfl_up_sync(FULL, ia, o), yb = __shfl_up_sync(FULL, ib, o);
      if (c.lane >= o) { ia += ya; ib += yb; }
    }
    if (c.lane < c.NW) { s->scand[c.lane][0] = ia - xa; s->scand[c.lane][1] = ib - xb; }
    if (c.lane == 31) { s->scand_total[0] = ia; s->scand_total[1] = ib; }
  }
  __syncthreads();
  a = s->scand[c.warp][0];
  b = s->scand[c.warp][1];
  *ta = s->scand_total[0];
  *tb = s->scand_total[1];
  __syncthreads();
}

// ------------------------------------------------------ AHP L1 (Eq. 9, R10) --
__device__ double ahp_cell64(double d, int rule) {
  if (rule == 0) return d > 0 ? d : (d < 0 ? 1.0 / (-d) : 1.0);
  return d > 0 ? 1.0 + d : (d < 0 ? 1.0 / (1.0 - d) : 1.0);
}
// criteria-level priority of the weights (one thread)
__device__ void ahp_l1_dev(const Opt& o, double L1[4]) {
  if (o.l1_mode == 1) {
    for (int c = 0; c < 4; ++c) L1[c] = o.wd[c];
    return;
  }
  double lo = o.wd[0], hi = o.wd[0];
  for (int c = 1; c < 4; ++c) { lo = fmin(lo, o.wd[c]); hi = fmax(hi, o.wd[c]); }
  if (hi == lo) {
    for (int c = 0; c < 4; ++c) L1[c] = 0.25;
    return;
  }
  double col[4];
  for (int j = 0; j < 4; ++j) {
    col[j] = 0;
    for (int i = 0; i < 4; ++i) col[j] += ahp_cell64(9.0 * (o.wd[i] - o.wd[j]) / (hi - lo), o.ahp_rule);
  }
  for (int i = 0; i < 4; ++i) {
    double a = 0;
    for (int j = 0; j < 4; ++j) a += ahp_cell64(9.0 * (o.wd[i] - o.wd[j]) / (hi - lo), o.ahp_rule) / col[j];
    L1[i] = a / 4.0;
  }
}

// ------------------------------------------------------------- fabric ------
// Widest ECMP path from server u to server v on the current residuals (R16),
// computed by warp 0; returns (path id, fabric bottleneck) in all lanes.
__device__ int2 widest_path_warp(Ctx& c, int u, int v) {
  const Geo& g = c.g;
  int h = g.h;
  int eu = (int)div_h(u, g.magic_h), ev = (int)div_h(v, g.magic_h);
  if (eu == ev) return make_int2(0, INT_MAX);
  int pu = (int)div_h(eu, g.magic_h), pv = (int)div_h(ev, g.magic_h);
  const int* EA = c.st + 4 * g.n;
  const int* AC = EA + g.E * h;
  int best = -1, bt = INT_MAX;
  if (pu == pv) {
    for (int a = c.lane; a < h; a += 32) {
      int b = min(EA[eu * h + a], EA[ev * h + a]);
      if (b > best) { best = b; bt = a; }
    }
  } else {
    for (int t = c.lane; t < h * h; t += 32) {
      int a = (int)div_h(t, g.magic_h), b = t - a * h;
      int x = min(min(EA[eu * h + a], EA[ev * h + a]), min(AC[(pu * h + a) * h + b], AC[(pv * h + a) * h + b]));
      if (x > best) { best = x; bt = t; }
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    int ob = __shfl_xor_sync(FULL, best, o);
    int ot = __shfl_xor_sync(FULL, bt, o);
    if (ob > best || (ob == best && ot < bt)) { best = ob; bt = ot; }
  }
  return make_int2(pu == pv ? 1 + bt : 1 + h + bt, best);
}

// Offsets of the fabric links of path `pid` between servers u and v; returns count.
__device__ int path_links(const Geo& g, int u, int v, int pid, int off[4]) {
  if (pid <= 0) return 0;
  int h = g.h;
  int eu = (int)div_h(u, g.magic_h), ev = (int)div_h(v, g.magic_h);
  int ea0 = 4 * g.n, ac0 = ea0 + g.E * h;
  if (pid <= h) {
    int a = pid - 1;
    off[0] = ea0 + eu * h + a;
    off[1] = ea0 + ev * h + a;
    return 2;
  }
  int t = pid - 1 - h;
  int a = (int)div_h(t, g.magic_h), b = t - a * h;
  int pu = (int)div_h(eu, g.magic_h), pv = (int)div_h(ev, g.magic_h);
  off[0] = ea0 + eu * h + a;
  off[1] = ac0 + (pu * h + a) * h + b;
  off[2] = ac0 + (pv * h + a) * h + b;
  off[3] = ea0 + ev * h + a;
  return 4;
}

// a2: mark edge switches from which some flow's widest fabric bottleneck is below its
// demand (SURVEY §8(a) a2 as threshold bitmasks).  All threads.
__device__ void fabric_tables(Ctx& c) {
  Scratch* s = c.s;
  const Geo& g = c.g;
  int h = g.h;
  const int* EA = c.st + 4 * g.n;
  const int* AC = EA + g.E * h;
  for (int f = 0; f < s->nflow; ++f) {
    int v = s->fv[f], D = s->fD[f];
    if (D <= s->minfab) continue;  // every fabric link carries D: no edge switch fails this flow
    int ev = (int)div_h(v, g.magic_h), pv = (int)div_h(ev, g.magic_h);
    for (int p = c.tid; p < g.k; p += c.B) s->pm[p] = 0u;
    if (c.tid == 0) s->vm = 0;
    __syncthreads();
    // pm[p] bit a: some core (a, b) links pod p and pod pv with both links >= D
    for (int t = c.tid; t < g.k * h; t += c.B) {
      int p = (int)div_h(t, g.magic_h), a = t - p * h;
      bool ok = false;
      const int* r1 = AC + (p * h + a) * h;
      const int* r2 = AC + (pv * h + a) * h;
      for (int b = 0; b < h && !ok; ++b) ok = r1[b] >= D && r2[b] >= D;
      if (ok) atomicOr(&s->pm[p], 1u << a);
    }
    for (int a = c.tid; a < h; a += c.B)
      if (EA[ev * h + a] >= D) atomicOr((unsigned*)&s->vm, 1u << a);
    __syncthreads();
    unsigned vm = (unsigned)s->vm;
    for (int e = c.tid; e < g.E; e += c.B) {
      if (e == ev) continue;  // same edge switch: access links only
      unsigned em = 0;
      for (int a = 0; a < h; ++a) em |= (EA[e * h + a] >= D ? 1u : 0u) << a;
      int pe = (int)div_h(e, g.magic_h);
      unsigned ok = (pe == pv) ? (em & vm) : (em & vm & s->pm[pe]);
      if (!ok) atomicOr(&c.edgebad[e >> 5], 1u << (e & 31));
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------- pass A -------
// a3 + a4: feasibility mask and statistics over F.  Writes maskw, s->nf, mn, mx, sq.
// GRID: the servers are spread over every CTA of the grid (the sharded engine's k_sh_filter);
// each CTA reduces in its own shared memory and combines into facc[11] with integer atomics
// (nf, nact, min/max of CPU, RAM, bandwidth, sums of squares — exact, order-independent);
// k_sh_prep_b then moves facc into the scratch fields.
// a4's reductions of pass_filter: per-thread statistics -> the CTA's (scratch) or, with GRID,
// the grid's (exact integer atomics into facc).  All threads.
template <bool GRID>
__device__ void filter_reduce(Ctx& c, int nf, int nact, unsigned mn0, unsigned mx0, unsigned mn1, unsigned mx1,
                              unsigned mn3, unsigned mx3, unsigned long long q0, unsigned long long q1,
                              unsigned long long q3, unsigned long long* facc) {
  __shared__ int g_red_i[GRID ? MAXW : 1][8];
  __shared__ unsigned long long g_red_u[GRID ? MAXW : 1][3];
  Scratch* s = c.s;
  // warp reductions (redux.sync for 32-bit, shuffles for 64-bit sums)
  nf = (int)__reduce_add_sync(FULL, (unsigned)nf);
  nact = (int)__reduce_add_sync(FULL, (unsigned)nact);
  mn0 = __reduce_min_sync(FULL, mn0); mx0 = __reduce_max_sync(FULL, mx0);
  mn1 = __reduce_min_sync(FULL, mn1); mx1 = __reduce_max_sync(FULL, mx1);
  mn3 = __reduce_min_sync(FULL, mn3); mx3 = __reduce_max_sync(FULL, mx3);
  for (int o = 16; o > 0; o >>= 1) {
    q0 += __shfl_xor_sync(FULL, q0, o);
    q1 += __shfl_xor_sync(FULL, q1, o);
    q3 += __shfl_xor_sync(FULL, q3, o);
  }
  int (*red_i)[8] = GRID ? g_red_i : s->red_i;
  unsigned long long (*red_u)[3] = GRID ? g_red_u : s->red_u;
  if (c.lane == 0) {
    int* r = red_i[c.warp];
    r[0] = nf; r[1] = nact; r[2] = (int)mn0; r[3] = (int)mx0; r[4] = (int)mn1; r[5] = (int)mx1;
    r[6] = (int)mn3; r[7] = (int)mx3;
    red_u[c.warp][0] = q0; red_u[c.warp][1] = q1; red_u[c.warp][2] = q3;
  }
  __syncthreads();
  if (c.warp == 0) {
    bool in = c.lane < c.NW;
    const int* r = red_i[in ? c.lane : 0];
    nf = in ? r[0] : 0; nact = in ? r[1] : 0;
    mn0 = in ? (unsigned)r[2] : UINT_MAX; mx0 = in ? (unsigned)r[3] : 0;
    mn1 = in ? (unsigned)r[4] : UINT_MAX; mx1 = in ? (unsigned)r[5] : 0;
    mn3 = in ? (unsigned)r[6] : UINT_MAX; mx3 = in ? (unsigned)r[7] : 0;
    q0 = in ? red_u[c.lane][0] : 0; q1 = in ? red_u[c.lane][1] : 0; q3 = in ? red_u[c.lane][2] : 0;
    nf = (int)__reduce_add_sync(FULL, (unsigned)nf);
    nact = (int)__reduce_add_sync(FULL, (unsigned)nact);
    mn0 = __reduce_min_sync(FULL, mn0); mx0 = __reduce_max_sync(FULL, mx0);
    mn1 = __reduce_min_sync(FULL, mn1); mx1 = __reduce_max_sync(FULL, mx1);
    mn3 = __reduce_min_sync(FULL, mn3); mx3 = __reduce_max_sync(FULL, mx3);
    for (int o = 16; o > 0; o >>= 1) {
      q0 += __shfl_xor_sync(FULL, q0, o);
      q1 += __shfl_xor_sync(FULL, q1, o);
      q3 += __shfl_xor_sync(FULL, q3, o);
    }
    if (GRID) {
      if (c.lane == 0) {
        atomicAdd(facc + 0, (unsigned long long)nf);
        atomicAdd(facc + 1, (unsigned long long)nact);
        atomicMin(facc + 2, (unsigned long long)mn0); atomicMax(facc + 3, (unsigned long long)mx0);
        atomicMin(facc + 4, (unsigned long long)mn1); atomicMax(facc + 5, (unsigned long long)mx1);
        atomicMin(facc + 6, (unsigned long long)mn3); atomicMax(facc + 7, (unsigned long long)mx3);
        atomicAdd(facc + 8, q0);
        atomicAdd(facc + 9, q1);
        atomicAdd(facc + 10, q3);
      }
    } else if (c.lane == 0) {
      s->nf = nf;
      s->nact = nact;
      s->mn[0] = (int)mn0; s->mx[0] = (int)mx0;
      s->mn[1] = (int)mn1; s->mx[1] = (int)mx1;
      s->mn[2] = nact == nf ? 1 : 0; s->mx[2] = nact > 0 ? 1 : 0;  // f_u in {0,1}
      s->mn[3] = (int)mn3; s->mx[3] = (int)mx3;
      s->sq[0] = q0; s->sq[1] = q1; s->sq[2] = (unsigned long long)nact; s->sq[3] = q3;
      s->c_feas += (unsigned long long)nf;
    }
  }
  __syncthreads();
}

template <bool WRITE_MASK, bool GRID = false>
__device__ void pass_filter(Ctx& c, uint8_t* mask_out, float* scores_out, unsigned long long* facc = nullptr) {
  Scratch* s = c.s;
  const Geo& g = c.g;
  const int n = g.n;
  const int* cpu = c.st;
  const int* ram = c.st + n;
  const int* act = c.st + 2 * n;
  const int* acc = c.st + 3 * n;     // access-link residuals: the filter (Eq. 5-7)
  const int* bwc = c.cr + 3 * n;     // the Bandwidth criterion (R2, or its logical reading)
  const int dc = s->dc, dr = s->dr, sumD = s->sumD;
  const bool net = c.o.path_filter && s->nflow > 0;
  const bool G = s->G != 0;
  int nf = 0, nact = 0;
  unsigned mn0 = UINT_MAX, mn1 = UINT_MAX, mn3 = UINT_MAX, mx0 = 0, mx1 = 0, mx3 = 0;
  unsigned long long q0 = 0, q1 = 0, q3 = 0;
  const int start = GRID ? (blockIdx.x * c.NW + c.warp) * 32 : c.warp * 32;
  const int stride = GRID ? gridDim.x * c.B : c.B;
  for (int base = start; base < n; base += stride) {
    int u = base + c.lane;
    bool in = u < n;
    int x0 = 0, x1 = 0, x2 = 0, x3 = 0;
    if (in) { x0 = cpu[u]; x1 = ram[u]; x2 = act[u]; x3 = bwc[u]; }
    bool ok = in && x0 >= dc && x1 >= dr;
    if (net) {
      unsigned e = div_h((unsigned)u, g.magic_h);
      ok = ok && G && acc[u] >= sumD && !((c.edgebad[e >> 5] >> (e & 31)) & 1u);
    }
    unsigned sp = c.special[base >> 5];
    if ((sp >> c.lane) & 1u) {
      // a flow server (its own flow needs no network) or an excluded server (R18)
      int f = -1;
      for (int i = 0; i < s->nflow; ++i) if (s->fv[i] == u) f = i;
      if (f < 0 || s->fexcl[f]) ok = false;
      else ok = x0 >= dc && x1 >= dr && (!c.o.path_filter || s->fok[f]);
    }
    unsigned bal = __ballot_sync(FULL, ok);
    if (c.lane == 0) c.maskw[base >> 5] = bal;
    if (WRITE_MASK && in) { mask_out[u] = ok ? 1 : 0; scores_out[u] = 0.0f; }
    if (ok) {
      nf += 1;
      nact += x2;
      mn0 = min(mn0, (unsigned)x0); mx0 = max(mx0, (unsigned)x0);
      mn1 = min(mn1, (unsigned)x1); mx1 = max(mx1, (unsigned)x1);
      mn3 = min(mn3, (unsigned)x3); mx3 = max(mx3, (unsigned)x3);
      q0 += (unsigned long long)((unsigned)x0) * (unsigned)x0;
      q1 += (unsigned long long)((unsigned)x1) * (unsigned)x1;
      q3 += (unsigned long long)((unsigned)x3) * (unsigned)x3;
    }
  }
  filter_reduce<GRID>(c, nf, nact, mn0, mx0, mn1, mx1, mn3, mx3, q0, q1, q3, facc);
}

// ------------------------------------------------------------ TOPSIS --------
// R25 walk: the best exact (FP64) score of the request's first pod step among the servers
// the current filter admits and that step admitted (scores in w64 + 2 n2, kept per request).
__device__ __forceinline__ double* rank_once_scores(const Ctx& c) {
  int n2 = 1;
  while (n2 < c.g.n) n2 <<= 1;
  return c.w64 + 2 * n2;  // after the AHP FP64 weights and level L2 (ahp_w64_doubles)
}
__device__ void rank_once_walk(Ctx& c) {
  const int n = c.g.n;
  const double* sc0 = rank_once_scores(c);
  double bv = -DBL_MAX;
  int bj = -1;
  for (int u = c.tid; u < n; u += c.B) {
    if (!(((c.maskw[u >> 5] & c.f0w[u >> 5]) >> (u & 31)) & 1u)) continue;
    const double v = sc0[u];
    if (v > bv || (v == bv && u < bj)) { bv = v; bj = u; }
  }
  block_argmax64(c, bv, bj);
}

template <bool WRITE_SCORES>
__device__ void select_topsis(Ctx& c, float* scores_out) {
  Scratch* s = c.s;
  const int n = c.g.n;
  const int* st = c.cr;  // criteria rows
  // R25: the first pod step ranks with its own statistics and keeps them with its feasible
  // set; later pod steps take the best of that order among the servers their filter admits
  if (c.o.rank_once && s->p > 0) {
    rank_once_walk(c);
    return;
  }
  TopsisP tp;
  for (int k = 0; k < 4; ++k) { tp.mx[k] = s->mx[k]; tp.mn[k] = s->mn[k]; }
  topsis_params(tp, c.o.wd, s->sq);
  if (c.o.rank_once) {  // keep the first pod step's feasible set and exact closeness
    double* sc0 = rank_once_scores(c);
    for (int w = c.tid; w < c.nW; w += c.B) c.f0w[w] = c.maskw[w];
    for (int u = c.tid; u < n; u += c.B)
      if ((c.maskw[u >> 5] >> (u & 31)) & 1u) sc0[u] = topsis64(tp, st[u], st[n + u], st[2 * n + u], st[3 * n + u]);
  }
  unsigned long long k1 = 0, k2 = 0;
  for (int base = c.warp * 32; base < n; base += c.B) {
    unsigned bits = c.maskw[base >> 5];
    if (!((bits >> c.lane) & 1u)) continue;
    int u = base + c.lane;
    float r = topsis32(tp, st[u], st[n + u], st[2 * n + u], st[3 * n + u]);
    if (WRITE_SCORES) scores_out[u] = r;
    top2_insert(k1, k2, score_key(r, u));
  }
  block_top2(c, k1, k2);
  if (c.tid == 0) {
    float s1 = __uint_as_float((unsigned)(s->key1 >> 32));
    float s2 = __uint_as_float((unsigned)(s->key2 >> 32));
    s->best = s->key1 ? (int)(0xFFFFFFFFu - (unsigned)(s->key1 & 0xFFFFFFFFull)) : -1;
    s->amb = s->key1 && (c.o.exact64 || (s->key2 != 0ull && s1 - s2 <= kTopsisDelta));
  }
  __syncthreads();
  if (s->amb) {  // FP64 re-decision over the near-max candidates (R14)
    float s1 = __uint_as_float((unsigned)(s->key1 >> 32));
    float thr = c.o.exact64 ? -1.0f : s1 - 2.0f * kTopsisDelta;
    double bv = -DBL_MAX;
    int bj = -1;
    for (int base = c.warp * 32; base < n; base += c.B) {
      unsigned bits = c.maskw[base >> 5];
      if (!((bits >> c.lane) & 1u)) continue;
      int u = base + c.lane;
      int x0 = st[u], x1 = st[n + u], x2 = st[2 * n + u], x3 = st[3 * n + u];
      if (topsis32(tp, x0, x1, x2, x3) < thr) continue;
      double r = topsis64(tp, x0, x1, x2, x3);
      if (r > bv || (r == bv && u < bj)) { bv = r; bj = u; }
    }
    block_argmax64(c, bv, bj);
    if (c.tid == 0) s->c_fp64 += 1;
  }
}

// ------------------------------------------------------------ BF / WF -------
// The orchestrators' native baselines ("BF (binpacking) and WF (spread)", reading
// R27): the feasible server (CPU/RAM filter: they "natively ignore the network
// requirements", routing follows at commit) of smallest (BF) or largest (WF) mean residual
// fraction (cpu/cpu_cap + ram/ram_cap) / 2, compared exactly as the integer
// cpu*ram_cap + ram*cpu_cap < 2^47; ties to the lowest index.  One packed 64-bit key per
// server, (key or its complement) << 17 | u, and a block-wide unsigned min.
template <bool WF>
__device__ void select_fit(Ctx& c) {
  Scratch* s = c.s;
  const int n = c.g.n;
  const int* st = c.st;
  constexpr unsigned long long KMAX = (1ull << 47) - 1;
  if (c.tid == 0) s->key1 = ~0ull;
  __syncthreads();
  unsigned long long best = ~0ull;
  for (int u = c.tid; u < n; u += c.B) {
    if (!((c.maskw[u >> 5] >> (u & 31)) & 1u)) continue;
    const unsigned long long key = (unsigned long long)st[u] * (unsigned)c.g.ram_cap +
                                   (unsigned long long)st[n + u] * (unsigned)c.g.cpu_cap;
    const unsigned long long k = WF ? KMAX - key : key;
    best = min(best, (k << 17) | (unsigned long long)u);
  }
  for (int o = 16; o; o >>= 1) best = min(best, __shfl_xor_sync(0xFFFFFFFFu, best, o));
  if (c.lane == 0 && best != ~0ull) atomicMin(&s->key1, best);
  __syncthreads();
  if (c.tid == 0) {
    s->best = s->key1 == ~0ull ? -1 : (int)(s->key1 & 0x1FFFFull);
    s->amb = 0;
  }
  __syncthreads();
}

// --------------------------------------------------------------- AHP --------
// a5A + a6A (Eq. 9-10, readings R7-R11).  Per criterion c with lo < hi over F,
// d_ij = s (x_i - x_j) with s = 9 / (hi - lo), a_ij = cell(d_ij), colsum_j = sum_i a_ij,
// L2_c[i] = (1/nf) sum_j a_ij / colsum_j, PG[i] = sum_c L1[c] L2_c[i].
//
// Sorted-level evaluation (no matrix, no compares).  The feasible values of c are sorted
// and collapsed into K levels v_0 < ... < v_{K-1} with multiplicities m_l.  A cell depends
// only on the two levels, so with the literal rule (R8: cell = d for d > 0, 1/(-d) for
// d < 0, 1 for d = 0):
//   colsum(l) = s * sum_{k>l} m_k (v_k - v_l) + m_l + (1/s) sum_{k<l} m_k / (v_l - v_k)
//   nf L2(l)  = s * sum_{k<l} w_k (v_l - v_k) + w_l + (1/s) sum_{k>l} w_k / (v_k - v_l),
// with w_k = m_k / colsum(k).  The linear sums come from exact double prefix sums; the
// reciprocal sums cost one reciprocal per unordered pair of levels per pass.  The shifted
// rule (1 + d, 1 / (1 - d)) adds the counts and uses 1 / (1 + s (v - v')).
__host__ __device__ inline int next_pow2(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}
// doubles of the FP64 re-decision workspace (per-level weights, per-level L2, priorities)
__host__ __device__ inline size_t ahp_w64_doubles(int n) { return 2 * (size_t)next_pow2(n) + (size_t)n; }
// bytes of the AHP workspace for n servers (ahp_carve layout)
__host__ __device__ inline size_t ahp_bytes(int n) {
  size_t n2 = (size_t)next_pow2(n);
  return align16(6 * n2) + align16(4 * (size_t)((n + 31) / 32)) + 2 * align16(4 * (size_t)n) + 4 * align16(4 * n2) +
         align16(4 * (n2 + 1)) + 2 * align16(8 * n2) + 2 * align16(8 * (n2 + 2)) + align16(4 * n2);
}
__device__ void ahp_carve(Ctx& c, unsigned char* base, int n) {
  size_t n2 = (size_t)next_pow2(n), off = 0;
  auto take = [&](size_t bytes) { unsigned char* p = base + off; off += align16(bytes); return p; };
  c.perm = reinterpret_cast<unsigned short*>(take(6 * n2));
  c.dirty = reinterpret_cast<unsigned*>(take(4 * (size_t)((n + 31) / 32)));
  c.pg = reinterpret_cast<float*>(take(4 * (size_t)n));
  c.lvl = reinterpret_cast<int*>(take(4 * (size_t)n));
  c.keys = reinterpret_cast<float*>(take(4 * n2));
  c.sidx = reinterpret_cast<int*>(take(4 * n2));
  c.keys2 = reinterpret_cast<float*>(take(4 * n2));
  c.sidx2 = reinterpret_cast<int*>(take(4 * n2));
  c.lst = reinterpret_cast<int*>(take(4 * (n2 + 1)));
  c.lvm = reinterpret_cast<float2*>(take(8 * n2));
  c.lvw = reinterpret_cast<float2*>(take(8 * n2));
  c.pa = reinterpret_cast<double*>(take(8 * (n2 + 2)));
  c.pb = reinterpret_cast<double*>(take(8 * (n2 + 2)));
  c.l2 = reinterpret_cast<float*>(take(4 * n2));
  c.nfcap = n;
}

// criterion index in the state (cpu 0, ram 1, access bandwidth 3) of presorted list ci
__device__ __forceinline__ int crit_of(int ci) { return ci == 2 ? 3 : ci; }

// Bitonic sort of keys[0..P2) ascending, payload sidx.  All threads.
__device__ void bitonic(Ctx& c, int P2) {
  for (int k = 2; k <= P2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = c.tid; i < P2; i += c.B) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const float a = c.keys[i], b = c.keys[ixj];
          if ((a > b) == ((i & k) == 0)) {
            c.keys[i] = b;
            c.keys[ixj] = a;
            const int t = c.sidx[i];
            c.sidx[i] = c.sidx[ixj];
            c.sidx[ixj] = t;
          }
        }
      }
      __syncthreads();
    }
  }
}

// Presort all servers by CPU, RAM and access bandwidth on the current state, and forget
// the dirty servers.  Once per snapshot (batch), per request (sequential), per query.
__device__ void ahp_presort(Ctx& c) {
  Scratch* s = c.s;
  const int n = c.g.n, P2 = next_pow2(n);
  for (int ci = 0; ci < 3; ++ci) {
    const int* x = c.cr + crit_of(ci) * n;
    for (int i = c.tid; i < P2; i += c.B) {
      c.keys[i] = i < n ? (float)x[i] : FLT_MAX;
      c.sidx[i] = i;
    }
    __syncthreads();
    bitonic(c, P2);
    for (int i = c.tid; i < n; i += c.B) c.perm[ci * P2 + i] = (unsigned short)c.sidx[i];
    __syncthreads();
  }
  for (int w = c.tid; w < c.nW; w += c.B) c.dirty[w] = 0u;
  if (c.tid == 0) { s->ntouched = 0; s->touch_over = 0; s->presorted = 1; }
  __syncthreads();
}

// Forget the servers the finished request touched (the state is the snapshot again).
__device__ void ahp_clear_dirty(Ctx& c) {
  Scratch* s = c.s;
  if (c.tid == 0) {
    const int nt = min(s->ntouched, 2 * MAXC);
    for (int i = 0; i < nt; ++i) {
      const int u = s->touched[i];
      c.dirty[u >> 5] &= ~(1u << (u & 31));
    }
    s->ntouched = 0;
  }
  __syncthreads();
}

// Levels of the m sorted values keys[0..m) (servers sidx): lvm[l] = (value, multiplicity),
// lvl[server] = level.  Returns K.  All threads (warp-segmented, coalesced).
__device__ int ahp_levels_sorted(Ctx& c, int m) {
  int s0, s1;
  warp_seg(c, m, s0, s1);
  int cnt = 0;
  for (int base = s0; base < s1; base += 32) {
    const int i = base + c.lane;
    const bool f = i < s1 && (i == 0 || c.keys[i] != c.keys[i - 1]);
    cnt += __popc(__ballot_sync(FULL, f));
  }
  int K;
  int l0 = warp_exscan(c, cnt, &K);
  for (int base = s0; base < s1; base += 32) {
    const int i = base + c.lane;
    const bool in = i < s1;
    const bool f = in && (i == 0 || c.keys[i] != c.keys[i - 1]);
    const unsigned bal = __ballot_sync(FULL, f);
    const int q = l0 + __popc(bal & (0xffffffffu >> (31 - c.lane))) - 1;  // level of element i
    if (f) {
      c.lvm[q].x = c.keys[i];
      c.lst[q] = i;
    }
    if (in) c.lvl[c.sidx[i]] = q;
    l0 += __popc(bal);
  }
  __syncthreads();
  for (int q = c.tid; q < K; q += c.B) c.lvm[q].y = (float)((q + 1 < K ? c.lst[q + 1] : m) - c.lst[q]);
  __syncthreads();
  return K;
}

__device__ __forceinline__ bool feas_bit(const Ctx& c, int u) { return (c.maskw[u >> 5] >> (u & 31)) & 1u; }

// Sorted values of presorted criterion ci into keys / sidx: walk the presorted order keeping
// the servers not touched by this request (only the feasible ones if feasible_only), then
// merge in the touched ones at their current values.  Returns the count.  All threads.
__device__ int presorted_collect(Ctx& c, int ci, bool feasible_only) {
  Scratch* s = c.s;
  const int n = c.g.n, P2 = next_pow2(n);
  const int* x = c.cr + crit_of(ci) * n;
  const unsigned short* perm = c.perm + ci * P2;
  int s0, s1;
  warp_seg(c, n, s0, s1);
  int cnt = 0;
  // unrolled: several independent gathers (perm -> value, feasibility, dirty) in flight
  // per warp when the arrays are in global memory (the sharded engine, 65536 servers)
#pragma unroll 4
  for (int base = s0; base < s1; base += 32) {
    const int i = base + c.lane;
    const int u = i < s1 ? perm[i] : 0;
    const bool k = i < s1 && (!feasible_only || feas_bit(c, u)) && !((c.dirty[u >> 5] >> (u & 31)) & 1u);
    cnt += __popc(__ballot_sync(FULL, k));
  }
  int mtot;
  int pos = warp_exscan(c, cnt, &mtot);
  if (c.tid == 0) s->m1 = mtot;
#pragma unroll 4
  for (int base = s0; base < s1; base += 32) {
    const int i = base + c.lane;
    const int u = i < s1 ? perm[i] : 0;
    const bool k = i < s1 && (!feasible_only || feas_bit(c, u)) && !((c.dirty[u >> 5] >> (u & 31)) & 1u);
    const unsigned bal = __ballot_sync(FULL, k);
    if (k) {
      const int q = pos + __popc(bal & ((1u << c.lane) - 1u));
      c.keys2[q] = (float)x[u];
      c.sidx2[q] = u;
    }
    pos += __popc(bal);
  }
  if (c.tid == 0) {  // touched servers, insertion-sorted by current value
    int d = 0;
    const int nt = min(s->ntouched, 2 * MAXC);
    for (int t = 0; t < nt; ++t) {
      const int u = s->touched[t];
      if (feasible_only && !feas_bit(c, u)) continue;
      const float v = (float)x[u];
      int j = d;
      while (j > 0 && s->dval[j - 1] > v) { s->dval[j] = s->dval[j - 1]; s->dsrv[j] = s->dsrv[j - 1]; --j; }
      s->dval[j] = v;
      s->dsrv[j] = u;
      ++d;
    }
    s->nd = d;
  }
  __syncthreads();
  const int m1 = s->m1, d = s->nd;
  for (int i = c.tid; i < m1; i += c.B) {  // untouched values shift past the touched ones below them
    const float v = c.keys2[i];
    int lo = 0, hi = d;
    while (lo < hi) { int mid = (lo + hi) >> 1; if (s->dval[mid] < v) lo = mid + 1; else hi = mid; }
    c.keys[i + lo] = v;
    c.sidx[i + lo] = c.sidx2[i];
  }
  for (int j = c.tid; j < d; j += c.B) {  // touched values after the untouched ones <= them
    const float v = s->dval[j];
    int lo = 0, hi = m1;
    while (lo < hi) { int mid = (lo + hi) >> 1; if (c.keys2[mid] <= v) lo = mid + 1; else hi = mid; }
    c.keys[j + lo] = v;
    c.sidx[j + lo] = s->dsrv[j];
  }
  __syncthreads();
  return m1 + d;
}

// Sorted feasible values of presorted criterion ci and their levels.  Returns K.
__device__ int ahp_levels_presorted(Ctx& c, int ci) {
  return ahp_levels_sorted(c, presorted_collect(c, ci, true));
}

// After an accepted request (sequential modes) the touched servers take their new values:
// re-merge them into the presorted orders instead of sorting again.
__device__ void ahp_presort_update(Ctx& c) {
  Scratch* s = c.s;
  if (s->touch_over) {  // more than the merge list holds: sort again at the next request
    __syncthreads();
    if (c.tid == 0) s->presorted = 0;
    __syncthreads();
    return;
  }
  const int n = c.g.n, P2 = next_pow2(n);
  for (int ci = 0; ci < 3; ++ci) {
    const int m = presorted_collect(c, ci, false);
    for (int i = c.tid; i < m; i += c.B) c.perm[ci * P2 + i] = (unsigned short)c.sidx[i];
    __syncthreads();
  }
  ahp_clear_dirty(c);
}

// Levels of the Fragmentation criterion f_u in {0,1}: no sort needed.
__device__ int ahp_levels_active(Ctx& c) {
  Scratch* s = c.s;
  const int n = c.g.n;
  const int nf = s->nf, nact = s->nact;
  const int K = (nact > 0) + (nact < nf);
  const int base = nact < nf ? 0 : 1;  // level of f_u = 0 is 0 when present
  for (int u = c.tid; u < n; u += c.B)
    if (feas_bit(c, u)) c.lvl[u] = c.st[2 * n + u] ? (nact < nf ? 1 : 0) : 0;
  if (c.tid == 0) {
    int l = 0;
    if (nact < nf) c.lvm[l++] = make_float2(0.0f, (float)(nf - nact));
    if (nact > 0) c.lvm[l++] = make_float2(1.0f, (float)nact);
  }
  (void)base;
  __syncthreads();
  return K;
}

// Exclusive prefix sums over K levels of (y, y * x) of lv[] into pa, pb (pa[K], pb[K]
// totals), in double, warp-segmented (fixed summation order for a given block size).
__device__ void ahp_prefix(Ctx& c, int K, const float2* lv) {
  int s0, s1;
  warp_seg(c, K, s0, s1);
  double ta = 0, tb = 0;
  for (int base = s0; base < s1; base += 32) {
    const int i = base + c.lane;
    if (i < s1) { const float2 e = lv[i]; ta += (double)e.y; tb += (double)e.y * (double)e.x; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) { ta += __shfl_xor_sync(FULL, ta, o); tb += __shfl_xor_sync(FULL, tb, o); }
  double TA, TB;
  warp_exscan_d2(c, ta, tb, &TA, &TB);
  double ra = ta, rb = tb;  // running exclusive prefix of this warp
  for (int base = s0; base < s1; base += 32) {
    const int i = base + c.lane;
    double a = 0, b = 0;
    if (i < s1) { const float2 e = lv[i]; a = (double)e.y; b = (double)e.y * (double)e.x; }
    double ia = a, ib = b;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double ya = __shfl_up_sync(FULL, ia, o), yb = __shfl_up_sync(FULL, ib, o);
      if (c.lane >= o) { ia += ya; ib += yb; }
    }
    if (i < s1) { c.pa[i] = ra + (ia - a); c.pb[i] = rb + (ib - b); }
    ra += __shfl_sync(FULL, ia, 31);
    rb += __shfl_sync(FULL, ib, 31);
  }
  if (c.tid == 0) { c.pa[K] = TA; c.pb[K] = TB; }
  __syncthreads();
}

// sum over k in [k0, k1) of arr[k].y / D(k), D = (v - arr[k].x) (pass 1, below) or
// (arr[k].x - v) (pass 2, above), or 1 + s * that under the shifted rule.  Terms in FP32
// with MUFU reciprocals, summed in chunks of 32 (four interleaved accumulators); the
// chunk sums accumulate in FP64, so the error does not grow with the number of levels.
template <bool ABOVE, int RULE>  // RULE a template parameter: no per-term selects for the literal rule
__device__ __forceinline__ double rsum_f32(const float2* arr, int k0, int k1, float v, float sc) {
  constexpr int rule = RULE;
  double outer = 0.0;
  int k = k0;
  float h0 = 0.f;
  for (; k < k1 && (k & 3); ++k) {  // head up to a multiple of 4
    const float2 o = arr[k];
    const float d = ABOVE ? o.x - v : v - o.x;
    h0 += o.y * rcp_approx(rule ? fmaf(sc, d, 1.0f) : d);
  }
  outer += (double)h0;
  // Chunks of 32 terms in 8 groups of 4 sharing ONE reciprocal: every term m_i / d_i is
  // positive (d_i >= 1, exact integer differences; 1 + s d >= 1 under the shifted rule),
  // so m0/d0 + m1/d1 + m2/d2 + m3/d3 = N / (d0 d1 d2 d3) with N = (m0 d1 + m1 d0) d2 d3 +
  // (m2 d3 + m3 d2) d0 d1 has no cancellation; |d| < 2^24 keeps the product < 2^96, inside
  // FP32 range.  One MUFU.RCP per 4 terms instead of 4 (MUFU runs 16/clk/SM, FP32 128):
  // the group costs 15 FP32-pipe ops + 1 MUFU; relative error <= 10u per group.
  for (; k + 32 <= k1; k += 32) {
    float a0 = 0.f, a1 = 0.f;
    const float4* q = reinterpret_cast<const float4*>(arr + k);
#pragma unroll
    for (int t = 0; t < 16; t += 2) {
      const float4 x = q[t], y = q[t + 1];  // levels k+2t .. k+2t+3
      float d0 = ABOVE ? x.x - v : v - x.x, d1 = ABOVE ? x.z - v : v - x.z;
      float d2 = ABOVE ? y.x - v : v - y.x, d3 = ABOVE ? y.z - v : v - y.z;
      if (rule) {
        d0 = fmaf(sc, d0, 1.0f);
        d1 = fmaf(sc, d1, 1.0f);
        d2 = fmaf(sc, d2, 1.0f);
        d3 = fmaf(sc, d3, 1.0f);
      }
      const float p01 = d0 * d1, p23 = d2 * d3;
      const float n01 = fmaf(x.y, d1, x.w * d0), n23 = fmaf(y.y, d3, y.w * d2);
      const float N = fmaf(n01, p23, n23 * p01);
      if (t & 2) a1 = fmaf(N, rcp_approx(p01 * p23), a1);
      else a0 = fmaf(N, rcp_approx(p01 * p23), a0);
    }
    outer += (double)(a0 + a1);
  }
  float t0 = 0.f;
  for (; k < k1; ++k) {
    const float2 o = arr[k];
    const float d = ABOVE ? o.x - v : v - o.x;
    t0 += o.y * rcp_approx(rule ? fmaf(sc, d, 1.0f) : d);
  }
  return outer + (double)t0;
}

// Warp-cooperative version for long level lists (grid passes): lane takes terms
// k0 + lane + 32 j, FP32 chunks of 32 terms per lane into an FP64 lane sum, then a
// fixed-order shuffle tree (deterministic).
template <bool ABOVE, int RULE>
__device__ __forceinline__ double rsum_warp(const float2* arr, int k0, int k1, float v, float sc, int lane) {
  constexpr int rule = RULE;
  double outer = 0.0;
  int k = k0 + lane;
  while (k < k1) {
    float a0 = 0.f, a1 = 0.f;
    int j = 0;
    // groups of 4 terms (k, k+32, k+64, k+96) sharing one reciprocal, as in rsum_f32
    for (; j < 32 && k + 96 < k1; j += 4, k += 128) {
      const float2 o0 = arr[k], o1 = arr[k + 32], o2 = arr[k + 64], o3 = arr[k + 96];
      float d0 = ABOVE ? o0.x - v : v - o0.x, d1 = ABOVE ? o1.x - v : v - o1.x;
      float d2 = ABOVE ? o2.x - v : v - o2.x, d3 = ABOVE ? o3.x - v : v - o3.x;
      if (rule) {
        d0 = fmaf(sc, d0, 1.0f);
        d1 = fmaf(sc, d1, 1.0f);
        d2 = fmaf(sc, d2, 1.0f);
        d3 = fmaf(sc, d3, 1.0f);
      }
      const float p01 = d0 * d1, p23 = d2 * d3;
      const float n01 = fmaf(o0.y, d1, o1.y * d0), n23 = fmaf(o2.y, d3, o3.y * d2);
      a0 = fmaf(fmaf(n01, p23, n23 * p01), rcp_approx(p01 * p23), a0);
    }
    for (; j < 32 && k + 32 < k1; j += 2, k += 64) {
      const float2 o = arr[k], p = arr[k + 32];
      const float d0 = ABOVE ? o.x - v : v - o.x, d1 = ABOVE ? p.x - v : v - p.x;
      a0 = fmaf(o.y, rcp_approx(rule ? fmaf(sc, d0, 1.0f) : d0), a0);
      a1 = fmaf(p.y, rcp_approx(rule ? fmaf(sc, d1, 1.0f) : d1), a1);
    }
    if (j < 32 && k < k1) {
      const float2 o = arr[k];
      const float d0 = ABOVE ? o.x - v : v - o.x;
      a0 = fmaf(o.y, rcp_approx(rule ? fmaf(sc, d0, 1.0f) : d0), a0);
      k += 32;
    }
    outer += (double)(a0 + a1);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) outer += __shfl_xor_sync(FULL, outer, o);
  return outer;
}

// FP32 passes over the K levels of criterion kc -> l2out[l] = L2 of level l.
// Each thread takes level pairs (l, K-1-l) so every pair holds K-1 terms per pass.
__device__ void ahp_passes_f32(Ctx& c, int kc, int K, int m, float* l2out) {
  Scratch* s = c.s;
  const int rule = c.o.ahp_rule;
  const double sd = s->ahp_scaled[kc];
  const float sc = (float)sd;
  const double inv_sd = 1.0 / sd;
  ahp_prefix(c, K, c.lvm);
  const double PAK = c.pa[K], PBK = c.pb[K];
  const int half = (K + 1) >> 1;
  for (int t = c.tid; t < half; t += c.B) {
    for (int side = 0; side < 2; ++side) {
      const int l = side ? K - 1 - t : t;
      if (side && l == t) break;
      const float2 me = c.lvm[l];
      const double rec = rule ? rsum_f32<false, 1>(c.lvm, 0, l, me.x, sc) : rsum_f32<false, 0>(c.lvm, 0, l, me.x, sc);
      const double cgt = PAK - c.pa[l + 1];
      const double G = (PBK - c.pb[l + 1]) - cgt * (double)me.x;  // sum_{k>l} m_k (v_k - v_l), exact
      const double col = rule ? cgt + sd * G + (double)me.y + (double)rec
                              : sd * G + (double)me.y + (double)rec * inv_sd;
      c.lvw[l] = make_float2(me.x, (float)((double)me.y / col));
    }
  }
  __syncthreads();
  ahp_prefix(c, K, c.lvw);
  for (int t = c.tid; t < half; t += c.B) {
    for (int side = 0; side < 2; ++side) {
      const int l = side ? K - 1 - t : t;
      if (side && l == t) break;
      const float2 me = c.lvw[l];
      const double rec = rule ? rsum_f32<true, 1>(c.lvw, l + 1, K, me.x, sc) : rsum_f32<true, 0>(c.lvw, l + 1, K, me.x, sc);
      const double lin = (double)me.x * c.pa[l] - c.pb[l];  // sum_{k<l} w_k (v_l - v_k)
      const double L = rule ? c.pa[l] + sd * lin + (double)me.y + (double)rec
                            : sd * lin + (double)me.y + (double)rec * inv_sd;
      l2out[l] = (float)(L / (double)m);
    }
  }
  __syncthreads();
}

// FP64 passes (the rare R14 re-decision): same formulation, IEEE reciprocals, exact
// prefix sums of the FP64 weights.  w64[0..K) holds the weights.
__device__ void ahp_passes_f64(Ctx& c, int kc, int K, int m, double* l2out) {
  Scratch* s = c.s;
  const int rule = c.o.ahp_rule;
  const double sd = s->ahp_scaled[kc];
  ahp_prefix(c, K, c.lvm);
  const double PAK = c.pa[K], PBK = c.pb[K];
  for (int l = c.tid; l < K; l += c.B) {
    const double vl = c.lvm[l].x, ml = c.lvm[l].y;
    double rec = 0;
    for (int k = 0; k < l; ++k) {
      const double d = vl - (double)c.lvm[k].x;
      rec += (double)c.lvm[k].y / (rule ? 1.0 + sd * d : d);
    }
    const double cgt = PAK - c.pa[l + 1];
    const double G = (PBK - c.pb[l + 1]) - cgt * vl;
    const double col = rule ? cgt + sd * G + ml + rec : sd * G + ml + rec / sd;
    c.w64[l] = ml / col;
  }
  __syncthreads();
  for (int l = c.tid; l < K; l += c.B) {
    const double vl = c.lvm[l].x;
    double rec = 0, a = 0, b = 0;
    for (int k = l + 1; k < K; ++k) {
      const double d = (double)c.lvm[k].x - vl;
      rec += c.w64[k] / (rule ? 1.0 + sd * d : d);
    }
    for (int q = 0; q < l; ++q) { a += c.w64[q]; b += c.w64[q] * (double)c.lvm[q].x; }
    const double lin = vl * a - b;
    const double L = rule ? a + sd * lin + c.w64[l] + rec : sd * lin + c.w64[l] + rec / sd;
    l2out[l] = L / (double)m;
  }
  __syncthreads();
}

// levels of criterion k (0 cpu, 1 ram, 2 active, 3 access bandwidth) over F
__device__ int ahp_levels_of(Ctx& c, int k) {
  Scratch* s = c.s;
  if (k == 2) return ahp_levels_active(c);
  if (s->touch_over) {  // more touched servers than the merge list holds: presort again
    ahp_presort(c);
    if (c.tid == 0) s->touch_over = 2;  // the snapshot order must be rebuilt after the request
    __syncthreads();
  }
  return ahp_levels_presorted(c, k == 3 ? 2 : k);
}

template <bool WRITE_SCORES>
__device__ void select_ahp(Ctx& c, float* scores_out) {
  Scratch* s = c.s;
  const int n = c.g.n;
  const int nf = s->nf;
  if (c.o.rank_once && s->p > 0) {  // R25: best FP64 priority of the first pod step, admitted now
    rank_once_walk(c);
    return;
  }
  if (c.o.rank_once)  // the first pod step keeps its feasible set and exact priorities
    for (int w = c.tid; w < c.nW; w += c.B) c.f0w[w] = c.maskw[w];
  for (int u = c.tid; u < n; u += c.B) c.pg[u] = 0.0f;
  if (c.tid == 0) {
    for (int k = 0; k < 4; ++k) {
      int lo = s->mn[k], hi = s->mx[k];
      s->ahp_const[k] = hi == lo;
      double sc = hi > lo ? 9.0 / (double)(hi - lo) : 0.0;
      s->ahp_scaled[k] = sc;
      s->ahp_scale[k] = (float)sc;
    }
  }
  __syncthreads();
  const float inv_nf = rcp_approx((float)nf);
  for (int k = 0; k < 4; ++k) {
    if (s->ahp_const[k]) {  // every value equal: L2 = 1/nf
      const float add = s->L1[k] * inv_nf;
      for (int u = c.tid; u < n; u += c.B) c.pg[u] += add;
      __syncthreads();
      continue;
    }
    const int K = ahp_levels_of(c, k);
    if (c.tid == 0) s->c_pairs += (unsigned long long)K * (unsigned long long)(K - 1) / 2;
    ahp_passes_f32(c, k, K, nf, c.l2);
    for (int u = c.tid; u < n; u += c.B)
      if (feas_bit(c, u)) c.pg[u] = fmaf(s->L1[k], c.l2[c.lvl[u]], c.pg[u]);
    __syncthreads();
  }
  unsigned long long k1 = 0, k2 = 0;
  for (int u = c.tid; u < n; u += c.B) {
    if (!feas_bit(c, u)) continue;
    const float pgv = c.pg[u];
    if (WRITE_SCORES) scores_out[u] = pgv;
    top2_insert(k1, k2, score_key(pgv, u));
  }
  block_top2(c, k1, k2);
  const float drel = ahp_delta_rel(nf);
  if (c.tid == 0) {
    float s1 = __uint_as_float((unsigned)(s->key1 >> 32));
    float s2 = __uint_as_float((unsigned)(s->key2 >> 32));
    s->best = (int)(0xFFFFFFFFu - (unsigned)(s->key1 & 0xFFFFFFFFull));
    s->amb = c.o.exact64 || c.o.rank_once || (s->key2 != 0ull && s2 >= s1 * (1.0f - drel));
  }
  __syncthreads();
  if (s->amb) {  // FP64 re-decision (R14): the same level formulation in double, all of F
    const int n2 = next_pow2(n);
    double* l2d = c.w64 + n2;      // w64: [n2] weights | [n2] L2 per level | [n] priorities
    double* pg64 = c.w64 + 2 * n2;
    for (int u = c.tid; u < n; u += c.B) pg64[u] = 0.0;
    __syncthreads();
    for (int k = 0; k < 4; ++k) {
      if (s->ahp_const[k]) {
        const double add = s->L1d[k] / (double)nf;
        for (int u = c.tid; u < n; u += c.B) pg64[u] += add;
        __syncthreads();
        continue;
      }
      const int K = ahp_levels_of(c, k);
      ahp_passes_f64(c, k, K, nf, l2d);
      for (int u = c.tid; u < n; u += c.B)
        if (feas_bit(c, u)) pg64[u] += s->L1d[k] * l2d[c.lvl[u]];
      __syncthreads();
    }
    double bv = -DBL_MAX;
    int bj = -1;
    for (int u = c.tid; u < n; u += c.B) {
      if (!feas_bit(c, u)) continue;
      const double v = pg64[u];
      if (v > bv || (v == bv && u < bj)) { bv = v; bj = u; }
    }
    block_argmax64(c, bv, bj);
    if (c.tid == 0) s->c_fp64 += 1;
  }
}

// ------------------------------------------------------------- request ------
// Build the flows of pod p (R17): every vlink between p and a placed pod q on server v
// adds bw^min to D_v; flows sorted by ascending v.  Thread 0.
// build_flows with the vlinks' global loads spread over a warp (lane e reads vlink e's
// endpoints and demand; lane 0 merges them in vlink order, as build_flows).  Warp 0.
__device__ void build_flows_warp(Ctx& c, const ReqsDev& R, int r, int p) {
  Scratch* s = c.s;
  const int v0 = R.voff[r];
  int nflow = 0, sumD = 0;
  for (int e0 = 0; e0 < s->nV; e0 += 32) {
    const int e = e0 + c.lane;
    int v = -1, D = 0;
    if (e < s->nV) {
      const int a = s->cpod[R.src[v0 + e]], b = s->cpod[R.dst[v0 + e]];
      int other = -1;
      if (a == p && b != p && s->pod_srv[b] >= 0) other = b;
      else if (b == p && a != p && s->pod_srv[a] >= 0) other = a;
      if (other >= 0) { v = s->pod_srv[other]; D = R.bw_min[v0 + e]; }
    }
    unsigned has = __ballot_sync(FULL, v >= 0);
    while (has) {
      const int l = __ffs(has) - 1;
      has &= has - 1;
      const int vv = __shfl_sync(FULL, v, l), DD = __shfl_sync(FULL, D, l);
      if (c.lane == 0) {
        int i = 0;
        while (i < nflow && s->fv[i] < vv) ++i;
        if (i < nflow && s->fv[i] == vv) {
          s->fD[i] += DD;
        } else {
          for (int t = nflow; t > i; --t) { s->fv[t] = s->fv[t - 1]; s->fD[t] = s->fD[t - 1]; }
          s->fv[i] = vv;
          s->fD[i] = DD;
          ++nflow;
        }
        sumD += DD;
      }
    }
  }
  if (c.lane == 0) {
    s->nflow = nflow;
    s->sumD = sumD;
  }
}

__device__ void build_flows(Ctx& c, const ReqsDev& R, int r, int p) {
  Scratch* s = c.s;
  int v0 = R.voff[r];
  int nflow = 0, sumD = 0;
  for (int e = 0; e < s->nV; ++e) {
    int a = s->cpod[R.src[v0 + e]], b = s->cpod[R.dst[v0 + e]];
    int other = -1;
    if (a == p && b != p && s->pod_srv[b] >= 0) other = b;
    else if (b == p && a != p && s->pod_srv[a] >= 0) other = a;
    if (other < 0) continue;
    int v = s->pod_srv[other], D = R.bw_min[v0 + e];
    int i = 0;
    while (i < nflow && s->fv[i] < v) ++i;
    if (i < nflow && s->fv[i] == v) {
      s->fD[i] += D;
    } else {
      for (int t = nflow; t > i; --t) { s->fv[t] = s->fv[t - 1]; s->fD[t] = s->fD[t - 1]; }
      s->fv[i] = v;
      s->fD[i] = D;
      ++nflow;
    }
    sumD += D;
  }
  s->nflow = nflow;
  s->sumD = sumD;
}

// Per-flow-server feasibility when u = v_f (its own flow uses the host bus) and the
// all-flows access check G.  All threads; after fabric_tables.
__device__ void flow_server_ok(Ctx& c) {
  Scratch* s = c.s;
  const int* acc = c.st + 3 * c.g.n;
  if (c.B >= MAXF) {  // one flow per thread: every access word loaded once, at the same time
    const int f = c.tid, nflow = s->nflow;
    int u = 0, au = 0, bad = 0;
    if (f < nflow) {
      u = s->fv[f];
      au = acc[u];
      bad = au < s->fD[f];
    }
    // flow f's server is feasible iff its access link carries the other flows and every other
    // flow's peer carries its own flow: no bad peer other than possibly f itself
    const int nbad = __syncthreads_count(bad);
    if (f < nflow) {
      bool ok = au >= s->sumD - s->fD[f] && (nbad == 0 || (nbad == 1 && bad));
      const unsigned e = div_h((unsigned)u, c.g.magic_h);
      if ((c.edgebad[e >> 5] >> (e & 31)) & 1u) ok = false;
      s->fok[f] = ok;
      s->fexcl[f] = 0;
      atomicOr(&c.special[u >> 5], 1u << (u & 31));
      if (c.spok && (ok || !c.o.path_filter)) atomicOr(&c.spok[u >> 5], 1u << (u & 31));
    }
    if (c.tid == 0) s->G = nbad == 0;
    return;
  }
  for (int f = c.tid; f < s->nflow; f += c.B) {
    int u = s->fv[f];
    bool ok = acc[u] >= s->sumD - s->fD[f];
    for (int h = 0; h < s->nflow; ++h)
      if (h != f && acc[s->fv[h]] < s->fD[h]) ok = false;
    unsigned e = div_h((unsigned)u, c.g.magic_h);
    if ((c.edgebad[e >> 5] >> (e & 31)) & 1u) ok = false;
    s->fok[f] = ok;
    s->fexcl[f] = 0;
    atomicOr(&c.special[u >> 5], 1u << (u & 31));
    if (c.spok && (ok || !c.o.path_filter)) atomicOr(&c.spok[u >> 5], 1u << (u & 31));
  }
  if (c.tid == 0) {
    int G = 1;
    for (int h = 0; h < s->nflow; ++h)
      if (acc[s->fv[h]] < s->fD[h]) G = 0;
    s->G = G;
  }
}

__device__ void clear_bitmaps(Ctx& c) {
  for (int w = c.tid; w < c.nW; w += c.B) c.special[w] = 0u;
  if (c.spok)
    for (int w = c.tid; w < c.nW; w += c.B) c.spok[w] = 0u;
  for (int w = c.tid; w < c.nEW; w += c.B) c.edgebad[w] = 0u;
}

// Commit of the chosen server for pod p (a8; Eq. 4-5, R16-R18).  Warp 0.
__device__ void commit(Ctx& c, const ReqsDev& R, int r, int p) {
  Scratch* s = c.s;
  const Geo& g = c.g;
  const int n = g.n;
  int u = s->best;
  if (c.lane == 0) {
    s->log_mark = s->log_n;
    st_set(c, u, c.st[u] - s->dc);
    st_set(c, n + u, c.st[n + u] - s->dr);
    st_set(c, 2 * n + u, 1);
  }
  __syncwarp();
  int fail = 0;
  for (int f = 0; f < s->nflow; ++f) {
    int v = s->fv[f], D = s->fD[f];
    if (v == u) {
      if (c.lane == 0) s->fpath[f] = -1;
      continue;
    }
    int2 wp = widest_path_warp(c, u, v);
    if (c.lane == 0) {
      int bott = min(min(c.st[3 * n + u], c.st[3 * n + v]), wp.y);
      if (bott < D) {
        fail = 1;
      } else {
        st_set(c, 3 * n + u, c.st[3 * n + u] - D);
        st_set(c, 3 * n + v, c.st[3 * n + v] - D);
        int off[4];
        int m = path_links(g, u, v, wp.x, off);
        for (int t = 0; t < m; ++t) st_set(c, off[t], c.st[off[t]] - D);
        s->fpath[f] = wp.x;
      }
    }
    fail = __shfl_sync(FULL, fail, 0);
    if (fail) break;
  }
  if (c.lane == 0) {
    if (fail) {  // R18: undo this pod's commit, exclude u, redo the pod step
      undo_to(c, s->log_mark);
      int f = -1;
      for (int i = 0; i < s->nflow; ++i) if (s->fv[i] == u) f = i;
      if (f >= 0) s->fexcl[f] = 1;
      c.special[u >> 5] |= 1u << (u & 31);
      s->fail = 1;
      s->c_retries += 1;
    } else {
      s->fail = 0;
      s->pod_srv[p] = u;
      int v0 = R.voff[r];
      for (int e = 0; e < s->nV; ++e) {
        int a = s->cpod[R.src[v0 + e]], b = s->cpod[R.dst[v0 + e]];
        int other = -1;
        if (a == p && b != p && b < p) other = b;
        else if (b == p && a != p && a < p) other = a;
        if (other < 0) continue;
        int v = s->pod_srv[other];
        int fp = -1;
        for (int i = 0; i < s->nflow; ++i) if (s->fv[i] == v) fp = s->fpath[i];
        s->vpath[e] = fp;
      }
    }
  }
}

// Widest ECMP path from u to v (R16) over the WHOLE CTA: one candidate (a, or (a, b)) per
// thread, a block-wide max of (bottleneck << 32 | ~candidate) keeps the lowest candidate on
// ties, as widest_path_warp.  Returns (path id, fabric bottleneck) in every thread.
__device__ int2 widest_path_cta(Ctx& c, int u, int v) {
  const Geo& g = c.g;
  const int h = g.h;
  const int eu = (int)div_h(u, g.magic_h), ev = (int)div_h(v, g.magic_h);
  if (eu == ev) return make_int2(0, INT_MAX);
  const int pu = (int)div_h(eu, g.magic_h), pv = (int)div_h(ev, g.magic_h);
  const int* EA = c.st + 4 * g.n;
  const int* AC = EA + g.E * h;
  const int nc = pu == pv ? h : h * h;
  unsigned long long key = 0;
  for (int t = c.tid; t < nc; t += c.B) {
    int x;
    if (pu == pv) {
      x = min(EA[eu * h + t], EA[ev * h + t]);
    } else {
      const int a = (int)div_h(t, g.magic_h), b = t - a * h;
      x = min(min(EA[eu * h + a], EA[ev * h + a]), min(AC[(pu * h + a) * h + b], AC[(pv * h + a) * h + b]));
    }
    const unsigned long long k = ((unsigned long long)(unsigned)x << 32) | (0xFFFFFFFFu - (unsigned)t);
    key = k > key ? k : key;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long b = __shfl_xor_sync(FULL, key, o);
    key = b > key ? b : key;
  }
  Scratch* s = c.s;
  __syncthreads();
  if (c.lane == 0) s->red_k[c.warp][0] = key;
  __syncthreads();
  if (c.warp == 0) {
    key = c.lane < c.NW ? s->red_k[c.lane][0] : 0ull;
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long b = __shfl_xor_sync(FULL, key, o);
      key = b > key ? b : key;
    }
    if (c.lane == 0) s->key1 = key;
  }
  __syncthreads();
  key = s->key1;
  const int bt = (int)(0xFFFFFFFFu - (unsigned)(key & 0xFFFFFFFFull));
  return make_int2(pu == pv ? 1 + bt : 1 + h + bt, (int)(key >> 32));
}

// commit (a8) with the widest paths searched by the whole CTA (k_seq_cluster's leader: the
// other CTAs wait at the next barrier, so the search latency is on the critical path).  Same
// state changes, undo log, R18 handling and outputs as commit().  All threads.
__device__ void commit_cta(Ctx& c, const ReqsDev& R, int r, int p) {
  Scratch* s = c.s;
  const Geo& g = c.g;
  const int n = g.n;
  const int u = s->best;
  if (c.warp == 0) {  // the server's three words read in parallel, applied by lane 0 (no AHP dirty list here)
    const int w = c.lane < 3 ? st_get(c, c.lane * n + u) : 0;
    const int x0 = __shfl_sync(FULL, w, 0), x1 = __shfl_sync(FULL, w, 1), x2 = __shfl_sync(FULL, w, 2);
    if (c.lane == 0) {
      s->log_mark = s->log_n;
      st_set_v(c, u, x0, x0 - s->dc);
      st_set_v(c, n + u, x1, x1 - s->dr);
      st_set_v(c, 2 * n + u, x2, 1);
      s->fail = 0;
    }
  }
  __syncthreads();
  SEQC_T(15);
  for (int f = 0; f < s->nflow; ++f) {
    const int v = s->fv[f], D = s->fD[f];
    if (v == u) {
      if (c.tid == 0) s->fpath[f] = -1;
      continue;
    }
    const int2 wp = widest_path_cta(c, u, v);  // ends with __syncthreads: earlier deductions seen
    SEQC_T(16);
    if (c.warp == 0) {  // the path's words (2 access + up to 4 fabric) read by lanes 0..5 at once
      int off[6];
      off[0] = 3 * n + u;
      off[1] = 3 * n + v;
      const int m = path_links(g, u, v, wp.x, off + 2);
      const int val = c.lane < 2 + m ? st_get(c, off[c.lane < 6 ? c.lane : 0]) : 0;
      int x[6];
#pragma unroll
      for (int i = 0; i < 6; ++i) x[i] = __shfl_sync(FULL, val, i);
      if (c.lane == 0) {
        const int bott = min(min(x[0], x[1]), wp.y);
        if (bott < D) {
          s->fail = 1;
        } else {
          for (int i = 0; i < 2 + m; ++i) st_set_v(c, off[i], x[i], x[i] - D);
          s->fpath[f] = wp.x;
        }
      }
    }
    __syncthreads();
    SEQC_T(17);
    if (s->fail) break;
  }
  if (c.tid == 0) {
    if (s->fail) {  // R18: undo this pod's commit, exclude u, redo the pod step
      undo_to(c, s->log_mark);
      int f = -1;
      for (int i = 0; i < s->nflow; ++i) if (s->fv[i] == u) f = i;
      if (f >= 0) s->fexcl[f] = 1;
      c.special[u >> 5] |= 1u << (u & 31);
      if (c.spok) c.spok[u >> 5] &= ~(1u << (u & 31));
      s->c_retries += 1;
    } else {
      s->pod_srv[p] = u;
    }
  }
  if (!s->fail && c.warp == 0) {  // each vlink of pod p to an earlier pod takes its flow's path (lanes)
    const int v0 = R.voff[r];
    for (int e = c.lane; e < s->nV; e += 32) {
      const int a = s->cpod[R.src[v0 + e]], b = s->cpod[R.dst[v0 + e]];
      int other = -1;
      if (a == p && b != p && b < p) other = b;
      else if (b == p && a != p && a < p) other = a;
      if (other < 0) continue;
      const int v = s->pod_srv[other];
      int fp = -1;
      for (int i = 0; i < s->nflow; ++i) if (s->fv[i] == v) fp = s->fpath[i];
      s->vpath[e] = fp;
    }
  }
}

// Outputs of a non-accepted request (status 0 or -1).  All threads.
__device__ void write_rejected(Ctx& c, const ReqsDev& R, const OutDev& O, int r, int status) {
  int c0 = R.coff[r], nC = R.coff[r + 1] - c0;
  int v0 = R.voff[r], nV = R.voff[r + 1] - v0;
  for (int i = c.tid; i < nC; i += c.B) {
    O.server[c0 + i] = -1;
    O.cpu_a[c0 + i] = 0;
    O.ram_a[c0 + i] = 0;
  }
  for (int e = c.tid; e < nV; e += c.B) {
    O.bw_a[v0 + e] = 0;
    O.path[v0 + e] = -1;
  }
  if (c.tid == 0) O.status[r] = status;
}

// One request (SURVEY §8(c) oracle algorithm, steps 1-3).  All threads.  On return the
// state holds the accepted placement (sequential) or is restored (batch: keep=false).
// Request start: validate (R24), pods and their demands.  Sets s->req_ok.  All threads.
template <int METHOD>
__device__ void req_begin(Ctx& c, const ReqsDev& R, int r, bool keep) {
  Scratch* s = c.s;
  if (c.tid == 0) {
    int c0 = R.coff[r], v0 = R.voff[r];
    int nC = R.coff[r + 1] - c0, nV = R.voff[r + 1] - v0;
    int bad = validate_request(nC, nV, R.cpu_min + c0, R.cpu_max + c0, R.ram_min + c0, R.ram_max + c0,
                               R.pod_of + c0, R.src + v0, R.dst + v0, R.bw_min + v0, R.bw_max + v0);
    s->req_ok = bad == 0;
    s->nC = nC;
    s->nV = nV;
    s->log_n = 0;
    if (bad) {
      s->c_invalid += 1;
    } else {
      int P = 0;
      for (int i = 0; i < nC; ++i) {
        int p = R.pod_of[c0 + i];
        s->cpod[i] = p;
        P = max(P, p + 1);
      }
      s->P = P;
      for (int p = 0; p < P; ++p) { s->pod_cpu[p] = 0; s->pod_ram[p] = 0; s->pod_srv[p] = -1; }
      for (int i = 0; i < nC; ++i) {
        s->pod_cpu[s->cpod[i]] += R.cpu_min[c0 + i];
        s->pod_ram[s->cpod[i]] += R.ram_min[c0 + i];
      }
      for (int e = 0; e < nV; ++e) s->vpath[e] = -1;
    }
  }
  __syncthreads();
  if (METHOD == 0) {  // presorted criteria: sort once, then keep the order (see ahp_presort_update)
    if (s->touch_over || !s->presorted) ahp_presort(c);
    else ahp_clear_dirty(c);
  }
}

// Pod p's prologue (a1, a2): demands, flows, fabric tables, flow-server feasibility.
__device__ void pod_prologue(Ctx& c, const ReqsDev& R, int r, int p) {
  Scratch* s = c.s;
  if (c.tid == 0) {
    s->p = p;
    s->dc = s->pod_cpu[p];
    s->dr = s->pod_ram[p];
  }
  SEQC_T(23);
  if (c.warp == 0) build_flows_warp(c, R, r, p);
  SEQC_T(22);
  clear_bitmaps(c);
  __syncthreads();
  SEQC_T(18);
  if (c.o.path_filter && s->nflow > 0) fabric_tables(c);
  SEQC_T(19);
  flow_server_ok(c);
  __syncthreads();
}

// R20: reject the whole request atomically.
__device__ void req_reject(Ctx& c, const ReqsDev& R, const OutDev& O, int r) {
  if (c.tid == 0) undo_to(c, 0);
  __syncthreads();
  write_rejected(c, R, O, r, 0);
  __syncthreads();
}

// a9: top-up (R19) in container order, then vlink order; emit the placement.
__device__ void req_finish(Ctx& c, const ReqsDev& R, const OutDev& O, int r, bool keep) {
  Scratch* s = c.s;
  const Geo& g = c.g;
  const int n = g.n;
  if (c.tid == 0) {
    int c0 = R.coff[r], v0 = R.voff[r];
    for (int i = 0; i < s->nC; ++i) {
      int u = s->pod_srv[s->cpod[i]];
      int cmin = R.cpu_min[c0 + i], rmin = R.ram_min[c0 + i];
      const int xc = st_get(c, u), xr = st_get(c, n + u);  // two independent loads
      int ec = min(R.cpu_max[c0 + i] - cmin, xc);
      int er = min(R.ram_max[c0 + i] - rmin, xr);
      if (ec) st_set_v(c, u, xc, xc - ec);
      if (er) st_set_v(c, n + u, xr, xr - er);
      O.server[c0 + i] = u;
      O.cpu_a[c0 + i] = cmin + ec;
      O.ram_a[c0 + i] = rmin + er;
    }
    for (int e = 0; e < s->nV; ++e) {
      int us = s->pod_srv[s->cpod[R.src[v0 + e]]], ud = s->pod_srv[s->cpod[R.dst[v0 + e]]];
      int bmin = R.bw_min[v0 + e], bmax = R.bw_max[v0 + e];
      if (us == ud) {
        O.bw_a[v0 + e] = bmax;
        O.path[v0 + e] = -1;
        continue;
      }
      int pid = s->vpath[e];
      int off[6];
      off[0] = 3 * n + us;
      off[1] = 3 * n + ud;
      const int m = 2 + path_links(g, us, ud, pid, off + 2);
      int x[6];  // the path's words, loaded together (distinct links: no reload after a store)
#pragma unroll
      for (int t = 0; t < 6; ++t) x[t] = t < m ? st_get(c, off[t]) : INT_MAX;
      int resid = x[0];
#pragma unroll
      for (int t = 1; t < 6; ++t) resid = min(resid, x[t]);
      int extra = min(bmax - bmin, resid);
      if (extra) {
        for (int t = 0; t < m; ++t) st_set_v(c, off[t], x[t], x[t] - extra);
      }
      O.bw_a[v0 + e] = bmin + extra;
      O.path[v0 + e] = pid;
    }
    O.status[r] = 1;
    if (!keep) undo_to(c, 0);
  }
  __syncthreads();
}

// One request (SURVEY §8(c) oracle algorithm, steps 1-3).  All threads.  On return the
// state holds the accepted placement (sequential) or is restored (batch: keep=false).
template <int METHOD>
__device__ void run_request(Ctx& c, const ReqsDev& R, const OutDev& O, int r, bool keep) {
  Scratch* s = c.s;
  req_begin<METHOD>(c, R, r, keep);
  if (!s->req_ok) {
    write_rejected(c, R, O, r, -1);
    __syncthreads();
    return;
  }
  const int P = s->P;
  for (int p = 0; p < P; ++p) {
    pod_prologue(c, R, r, p);
    for (;;) {
      pass_filter<false>(c, nullptr, nullptr);
      if (c.tid == 0) s->c_steps += 1;
      if (s->nf == 0) {
        req_reject(c, R, O, r);
        return;
      }
      if (METHOD == 1) select_topsis<false>(c, nullptr);
      else if (METHOD == 0) select_ahp<false>(c, nullptr);
      else select_fit<METHOD == 3>(c);
      if (s->best < 0) {  // R25: no server of the request's order is admitted (R20)
        req_reject(c, R, O, r);
        return;
      }
      if (c.warp == 0) commit(c, R, r, p);
      __syncthreads();
      if (!s->fail) break;
    }
  }
  req_finish(c, R, O, r, keep);
  if (METHOD == 0 && keep) ahp_presort_update(c);
}

// ------------------------------------------------------------- kernels ------
__device__ void ctx_basic(Ctx& c, const Geo& g, const Opt& o, Scratch* s) {
  c.g = g;
  c.o = o;
  c.s = s;
  c.tid = threadIdx.x;
  c.B = blockDim.x;
  c.NW = blockDim.x >> 5;
  c.lane = threadIdx.x & 31;
  c.warp = threadIdx.x >> 5;
  c.nW = (g.n + 31) >> 5;
  c.nEW = (g.E + 31) >> 5;
  c.dirty = nullptr;
}

__device__ void init_ctx(Ctx& c, const Geo& g, const Opt& o, Scratch* s) {
  c.g = g;
  c.o = o;
  c.s = s;
  c.tid = threadIdx.x;
  c.B = blockDim.x;
  c.NW = blockDim.x >> 5;
  c.lane = threadIdx.x & 31;
  c.warp = threadIdx.x >> 5;
  c.nW = (g.n + 31) >> 5;
  c.nEW = (g.E + 31) >> 5;
  c.dirty = nullptr;
  c.mirr = nullptr;
  if (c.tid == 0) {
    s->c_steps = s->c_retries = s->c_fp64 = s->c_invalid = s->c_feas = s->c_pairs = 0;
    s->minfab = s->minfab0 = 0;
    s->presorted = 0;
    s->touch_over = 0;
    s->ntouched = 0;
    if (o.method == 0) {
      double L1[4];
      ahp_l1_dev(o, L1);
      for (int k = 0; k < 4; ++k) { s->L1d[k] = L1[k]; s->L1[k] = (float)L1[k]; }
    }
  }
}

__device__ void flush_stats(Ctx& c, unsigned long long* stats) {
  if (c.tid == 0) {
    Scratch* s = c.s;
    if (s->c_steps) atomicAdd(&stats[ST_POD_STEPS], s->c_steps);
    if (s->c_retries) atomicAdd(&stats[ST_RETRIES], s->c_retries);
    if (s->c_fp64) atomicAdd(&stats[ST_FP64], s->c_fp64);
    if (s->c_invalid) atomicAdd(&stats[ST_INVALID], s->c_invalid);
    if (s->c_feas) atomicAdd(&stats[ST_FEAS], s->c_feas);
    if (s->c_pairs) atomicAdd(&stats[ST_PAIRS], s->c_pairs);
  }
}

// s->minfab = the smallest fabric residual of the state (block reduction).  All threads.
__device__ void init_minfab(Ctx& c) {
  const int n = c.g.n, L = c.g.L;
  int m = INT_MAX;
  for (int i = 4 * n + c.tid; i < 3 * n + L; i += c.B) m = min(m, c.st[i]);
  m = (int)__reduce_min_sync(FULL, (unsigned)m);  // residuals are >= 0
  if (c.lane == 0) c.s->red_i[c.warp][0] = m;
  __syncthreads();
  if (c.tid == 0) {
    int b = INT_MAX;
    for (int w = 0; w < c.NW; ++w) b = min(b, c.s->red_i[w][0]);
    c.s->minfab = c.s->minfab0 = b == INT_MAX ? 0 : b;
  }
  __syncthreads();
}

// dynamic shared memory layout of k_batch:
//   state words (6n ints) | maskw[nW] | special[nW] | edgebad[nEW] | AHP arrays

template <int METHOD, bool AHPG = false>
__global__ void __launch_bounds__(1024) k_batch(Geo g, Opt o, const int* __restrict__ snap, ReqsDev R,
                                                OutDev O, int2* ulog, double* w64, unsigned char* ahp_g, int* next,
                                                unsigned long long* stats, const int* idx, const int* n_idx) {
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ Scratch s;
  __shared__ __align__(8) unsigned long long mbar;
  const int n_req = idx ? *n_idx : R.n;  // deferred list from k_batch_warp, or every request
  if (n_req == 0) return;
  Ctx c;
  init_ctx(c, g, o, &s);
  const int nW = c.nW, nEW = c.nEW, n = g.n;
  size_t off = 0;
  c.st = reinterpret_cast<int*>(dyn);
  c.cr = c.st;
  off = align16(off + sizeof(int) * (size_t)g.words());
  c.maskw = reinterpret_cast<unsigned*>(dyn + off);
  off = align16(off + sizeof(unsigned) * nW);
  c.special = reinterpret_cast<unsigned*>(dyn + off);
  off = align16(off + sizeof(unsigned) * nW);
  c.f0w = reinterpret_cast<unsigned*>(dyn + off);
  off = align16(off + sizeof(unsigned) * nW);
  c.edgebad = reinterpret_cast<unsigned*>(dyn + off);
  off = align16(off + sizeof(unsigned) * nEW);
  c.nfcap = n;
  // (separate instantiations keep the shared-memory layout's pointers provably shared)
  if (METHOD == 0) ahp_carve(c, AHPG ? ahp_g + (size_t)blockIdx.x * align16(ahp_bytes(n)) : dyn + off, n);
  if (w64) c.w64 = w64 + (size_t)blockIdx.x * ahp_w64_doubles(n);  // AHP FP64; R25 scores
  c.snap = snap;
  c.ulog = ulog + (size_t)blockIdx.x * ULOG_CAP;

  // a0: the snapshot into shared memory with TMA bulk copies (cp.async.bulk).
  const unsigned bytes = (unsigned)(sizeof(int) * (size_t)g.words());  // 24 n, a multiple of 16
  if (c.tid == 0) {
    unsigned mb = smem_u32(&mbar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
    const unsigned chunk = 32768;
    for (unsigned o2 = 0; o2 < bytes; o2 += chunk) {
      unsigned sz = bytes - o2 < chunk ? bytes - o2 : chunk;
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(dyn + o2)),
          "l"(reinterpret_cast<const unsigned char*>(snap) + o2), "r"(sz), "r"(mb)
          : "memory");
    }
  }
  __syncthreads();
  {
    unsigned mb = smem_u32(&mbar);
    asm volatile(
        "{\n .reg .pred P1;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
        " @!P1 bra WAIT_%=;\n}" ::"r"(mb)
        : "memory");
  }
  for (int w = c.tid; w < nW; w += c.B) { c.maskw[w] = 0u; c.special[w] = 0u; }
  for (int w = c.tid; w < nEW; w += c.B) c.edgebad[w] = 0u;
  __syncthreads();
  init_minfab(c);
  if (METHOD == 0) ahp_presort(c);  // the snapshot's order serves every request

  for (;;) {
    if (c.tid == 0) s.next_req = atomicAdd(next, 1);
    __syncthreads();
    int r = s.next_req;
    __syncthreads();
    if (r >= n_req) break;
    if (idx) r = idx[r];
    run_request<METHOD>(c, R, O, r, false);
    if (c.tid == 0) s.minfab = s.minfab0;  // the request's overlay is undone: the snapshot again
  }
  flush_stats(c, stats);
}

// Sequential kernels keep the live state in shared memory when it fits (k <= 32 with the
// bitmaps: every serial step of a pod step — flows, commit, top-up — then reads on-chip
// words instead of L2), copied in at the start and back at the end of the launch.
__device__ int* load_state_smem(Ctx& c, unsigned char* base, const int* state) {
  int* sst = reinterpret_cast<int*>(base);
  const int W = c.g.words();
  for (int i = c.tid; i < W; i += c.B) sst[i] = state[i];
  __syncthreads();
  return sst;
}
__device__ void store_state_smem(Ctx& c, const int* sst, int* state) {
  __syncthreads();
  const int W = c.g.words();
  for (int i = c.tid; i < W; i += c.B) state[i] = sst[i];
}

template <int METHOD>
__global__ void __launch_bounds__(1024) k_sequential(Geo g, Opt o, int* state, ReqsDev R, OutDev O, int2* ulog,
                                                     float* ahp_ws, double* w64, unsigned long long* stats,
                                                     int smem_state) {
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ Scratch s;
  Ctx c;
  init_ctx(c, g, o, &s);
  size_t off = 0;
  c.maskw = reinterpret_cast<unsigned*>(dyn + off);
  off = align16(off + sizeof(unsigned) * c.nW);
  c.special = reinterpret_cast<unsigned*>(dyn + off);
  off = align16(off + sizeof(unsigned) * c.nW);
  c.f0w = reinterpret_cast<unsigned*>(dyn + off);
  off = align16(off + sizeof(unsigned) * c.nW);
  c.edgebad = reinterpret_cast<unsigned*>(dyn + off);
  off = align16(off + sizeof(unsigned) * c.nEW);
  int* sst = smem_state ? load_state_smem(c, dyn + off, state) : state;
  c.st = sst;
  c.cr = c.st;
  c.snap = sst;
  c.ulog = ulog;
  c.nfcap = g.n;
  if (METHOD == 0) ahp_carve(c, reinterpret_cast<unsigned char*>(ahp_ws), g.n);
  c.w64 = w64;
  for (int w = c.tid; w < c.nW; w += c.B) { c.maskw[w] = 0u; c.special[w] = 0u; }
  for (int w = c.tid; w < c.nEW; w += c.B) c.edgebad[w] = 0u;
  __syncthreads();
  init_minfab(c);
  for (int r = 0; r < R.n; ++r) run_request<METHOD>(c, R, O, r, true);
  if (smem_state) store_state_smem(c, sst, state);
  flush_stats(c, stats);
}

// ------------------------------------------- sequential engine on a cluster ---
// nacs_schedule_request for TOPSIS on a large DC (the paper's online semantics, P:206, P:391,
// on C5's 65536 servers): ONE thread-block cluster of C CTAs runs the whole request stream in
// one launch, no host round trip.  Every CTA keeps its own scratch (request decode, pods,
// flows, fabric tables, flow-server feasibility: identical, deterministic copies) and filters
// and scores its grid-stride share of the servers on the live state in global memory (L2);
// the exact integer statistics meet in global accumulators (atomics, double-buffered per
// attempt), the top-2 keys (and FP64 near-tie candidates) in one slot per CTA.  The leader
// (rank 0) alone commits (a8, R16-R18), tops up (R19), rejects (R20) and writes outputs; the
// others read its verdict (R18 failure) and fabric bound over DSMEM after the barrier and
// replicate the exclusion.  Three cluster barriers per pod step.
namespace cgx = cooperative_groups;

__device__ __forceinline__ void facc_reset(unsigned long long* f, int tid) {
  if (tid < 11) f[tid] = (tid >= 2 && tid <= 7 && !(tid & 1)) ? ~0ull : 0ull;
}


// k_seq_cluster's a3 + a4: pass_filter's test on this CTA's grid-stride share of at most
// SQ_J servers per thread, read from the CTA's shared-memory copy of the rows (mir; the
// cluster lives in one GPC, whose L2 port made the 1 MB global read of every pod step the
// largest phase) and kept in registers for the scoring pass.
__device__ __forceinline__ void seqc_filter(Ctx& c, const int* mir, unsigned long long* facc, unsigned& okb) {
  SEQC_T(21);
  Scratch* s = c.s;
  const Geo& g = c.g;
  const int n = g.n;
  const int dc = s->dc, dr = s->dr, sumD = s->sumD;
  const bool net = c.o.path_filter && s->nflow > 0;
  const bool G = s->G != 0;
  const int start = (blockIdx.x * (SQC_T >> 5) + c.warp) * 32, stride = gridDim.x * SQC_T;
  int x[SQ_J][4];
#pragma unroll
  for (int j = 0; j < SQ_J; ++j) {
    const int u = start + j * stride + c.lane;
    const bool in = u < n;
#pragma unroll
    for (int q = 0; q < 4; ++q) x[j][q] = in ? mir[q * SQC_M + j * SQC_T + c.tid] : 0;
  }
#ifdef NACS_SEQC_PROF
  asm volatile("" ::"r"(x[0][0]), "r"(x[SQ_J - 1][3]));
#endif
  SEQC_T(20);
  int nf = 0, nact = 0;
  unsigned mn0 = UINT_MAX, mn1 = UINT_MAX, mn3 = UINT_MAX, mx0 = 0, mx1 = 0, mx3 = 0;
  unsigned long long q0 = 0, q1 = 0, q3 = 0;
  okb = 0;
  // the bitmap words of every share first (independent loads), then branch-free tests
  unsigned eb[SQ_J], sp[SQ_J], so[SQ_J];
#pragma unroll
  for (int j = 0; j < SQ_J; ++j) {
    const int base = start + j * stride;
    const int w = base < n ? base >> 5 : 0;
    const unsigned e = div_h((unsigned)min(base + c.lane, n - 1), g.magic_h);
    eb[j] = net ? c.edgebad[e >> 5] >> (e & 31) : 0u;
    sp[j] = c.special[w] >> c.lane;
    so[j] = c.spok[w] >> c.lane;
  }
#pragma unroll
  for (int j = 0; j < SQ_J; ++j) {
    const int base = start + j * stride;
    if (base >= n) break;  // warp-uniform
    const bool in = base + c.lane < n;
    const int x0 = x[j][0], x1 = x[j][1], x2 = x[j][2], x3 = x[j][3];
    const bool okr = in & (x0 >= dc) & (x1 >= dr);
    // a flow server (its own flow needs no network) or an excluded one (R18): the verdict
    // flow_server_ok and the exclusions keep in spok
    const bool ok = (sp[j] & 1u) ? okr & ((so[j] & 1u) != 0u)
                                 : okr & (!net | (G & (x3 >= sumD) & !(eb[j] & 1u)));
    const unsigned bal = __ballot_sync(FULL, ok);
    if (c.lane == 0) c.maskw[base >> 5] = bal;
    okb |= (ok ? 1u : 0u) << j;
    if (ok) {
      nf += 1;
      nact += x2;
      mn0 = min(mn0, (unsigned)x0); mx0 = max(mx0, (unsigned)x0);
      mn1 = min(mn1, (unsigned)x1); mx1 = max(mx1, (unsigned)x1);
      mn3 = min(mn3, (unsigned)x3); mx3 = max(mx3, (unsigned)x3);
      q0 += (unsigned long long)((unsigned)x0) * (unsigned)x0;
      q1 += (unsigned long long)((unsigned)x1) * (unsigned)x1;
      q3 += (unsigned long long)((unsigned)x3) * (unsigned)x3;
    }
  }
  SEQC_T(10);
  filter_reduce<true>(c, nf, nact, mn0, mx0, mn1, mx1, mn3, mx3, q0, q1, q3, facc);
}

__global__ void __launch_bounds__(SQC_T, 1) k_seq_cluster(Geo g, Opt o, int* state, ReqsDev R, OutDev O, int2* ulog,
                                                      unsigned long long* stats, unsigned long long* facc,
                                                      unsigned long long* kx, double* kxv, int* kxi) {
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ Scratch s;
  cgx::cluster_group cl = cgx::this_cluster();
  const int C = (int)cl.num_blocks(), q = (int)cl.block_rank();
  const bool lead = q == 0;
  Ctx c;
  init_ctx(c, g, o, &s);
  c.B = SQC_T;  // compile-time block shape: the compiler folds it instead of re-deriving it
  c.NW = SQC_T >> 5;
  size_t off = 0;
  c.maskw = reinterpret_cast<unsigned*>(dyn + off);
  off = align16(off + sizeof(unsigned) * c.nW);
  c.special = reinterpret_cast<unsigned*>(dyn + off);
  off = align16(off + sizeof(unsigned) * c.nW);
  c.f0w = reinterpret_cast<unsigned*>(dyn + off);
  off = align16(off + sizeof(unsigned) * c.nW);
  c.edgebad = reinterpret_cast<unsigned*>(dyn + off);
  off = align16(off + sizeof(unsigned) * c.nEW);
  c.spok = reinterpret_cast<unsigned*>(dyn + off);
  off = align16(off + sizeof(unsigned) * c.nW);
  int* mir = reinterpret_cast<int*>(dyn + off);  // [4][SQC_M] this CTA's rows
  NACS_DCHECK(C * SQC_M >= g.n && (int)blockDim.x == SQC_T);
  __shared__ int* mirr[16];
  if (c.tid < C) mirr[c.tid] = cl.map_shared_rank(mir, c.tid);
  c.mirr = mirr;
  c.st = state;
  c.cr = state;
  c.snap = state;
  c.ulog = ulog;
  c.nfcap = g.n;
  c.w64 = nullptr;
  const int n = g.n;
#pragma unroll
  for (int j = 0; j < SQ_J; ++j) {
    const int u = blockIdx.x * SQC_T + j * C * SQC_T + c.tid;
#pragma unroll
    for (int q = 0; q < 4; ++q) mir[q * SQC_M + j * SQC_T + c.tid] = u < n ? state[q * n + u] : 0;
  }
  for (int w = c.tid; w < c.nW; w += c.B) { c.maskw[w] = 0u; c.special[w] = 0u; c.spok[w] = 0u; }
  for (int w = c.tid; w < c.nEW; w += c.B) c.edgebad[w] = 0u;
  if (lead) { facc_reset(facc, c.tid); facc_reset(facc + 16, c.tid); }
  __syncthreads();
  init_minfab(c);  // every CTA reads the same state: the same bound
  cl.sync();
  int t = 0;  // attempt counter (the same in every CTA)
#ifdef NACS_SEQC_PROF
  if (c.tid < 24) seqc_prof_[c.tid] = 0;
  if (c.tid == 0) seqc_last_ = SEQC_CLOCK();
#endif
  // the current request's arrays in shared memory (one parallel copy per request: the
  // thread-0 loops of decode, flows, commit and top-up then read on-chip), presented to the
  // device functions as a one-request batch (r = 0) with offset output pointers
  __shared__ int rq[5 * MAXC + 4 * MAXV];
  __shared__ int roff[4];
  for (int rg = 0; rg < R.n; ++rg) {
    const int c0 = R.coff[rg], nC = R.coff[rg + 1] - c0, v0 = R.voff[rg], nV = R.voff[rg + 1] - v0;
    const bool local = nC >= 0 && nC <= MAXC && nV >= 0 && nV <= MAXV;
    ReqsDev RL = R;
    OutDev OL = O;
    int r = rg;
    if (local) {
      for (int i = c.tid; i < nC; i += c.B) {
        rq[i] = R.cpu_min[c0 + i];
        rq[MAXC + i] = R.cpu_max[c0 + i];
        rq[2 * MAXC + i] = R.ram_min[c0 + i];
        rq[3 * MAXC + i] = R.ram_max[c0 + i];
        rq[4 * MAXC + i] = R.pod_of[c0 + i];
      }
      for (int e = c.tid; e < nV; e += c.B) {
        rq[5 * MAXC + e] = R.src[v0 + e];
        rq[5 * MAXC + MAXV + e] = R.dst[v0 + e];
        rq[5 * MAXC + 2 * MAXV + e] = R.bw_min[v0 + e];
        rq[5 * MAXC + 3 * MAXV + e] = R.bw_max[v0 + e];
      }
      if (c.tid == 0) { roff[0] = 0; roff[1] = nC; roff[2] = 0; roff[3] = nV; }
      RL.n = 1;
      RL.coff = roff;
      RL.voff = roff + 2;
      RL.cpu_min = rq;
      RL.cpu_max = rq + MAXC;
      RL.ram_min = rq + 2 * MAXC;
      RL.ram_max = rq + 3 * MAXC;
      RL.pod_of = rq + 4 * MAXC;
      RL.src = rq + 5 * MAXC;
      RL.dst = rq + 5 * MAXC + MAXV;
      RL.bw_min = rq + 5 * MAXC + 2 * MAXV;
      RL.bw_max = rq + 5 * MAXC + 3 * MAXV;
      OL.status = O.status + rg;
      OL.server = O.server + c0;
      OL.cpu_a = O.cpu_a + c0;
      OL.ram_a = O.ram_a + c0;
      OL.bw_a = O.bw_a + v0;
      OL.path = O.path + v0;
      r = 0;
      __syncthreads();
    }
    SEQC_T(0);
    req_begin<1>(c, RL, r, true);
    SEQC_T(1);
    if (!s.req_ok) {
      if (lead) write_rejected(c, RL, OL, r, -1);
      __syncthreads();  // the shared request copy is rewritten by the next request
      continue;
    }
    bool rejected = false;
    for (int p = 0; p < s.P && !rejected; ++p) {
      pod_prologue(c, RL, r, p);
      SEQC_T(2);
      for (;;) {
        unsigned long long* fa = facc + 16 * (t & 1);
        unsigned okb;
        seqc_filter(c, mir, fa, okb);  // a3 + a4 on this CTA's grid-stride share (rows kept in registers)
        SEQC_T(3);
        cl.sync();  // (1) the exact statistics of every CTA are in fa
        SEQC_T(4);
        if (c.warp == 0) {  // the 11 accumulators in one parallel load
          const unsigned long long fv = c.lane < 11 ? fa[c.lane] : 0ull;
          unsigned long long f[11];
#pragma unroll
          for (int i = 0; i < 11; ++i) f[i] = __shfl_sync(FULL, fv, i);
          if (c.lane == 0) {
            const int nf = (int)f[0], nact = (int)f[1];
            s.nf = nf;
            s.nact = nact;
            s.mn[0] = (int)f[2]; s.mx[0] = (int)f[3];
            s.mn[1] = (int)f[4]; s.mx[1] = (int)f[5];
            s.mn[2] = nact == nf ? 1 : 0; s.mx[2] = nact > 0 ? 1 : 0;  // f_u in {0,1}
            s.mn[3] = (int)f[6]; s.mx[3] = (int)f[7];
            s.sq[0] = f[8]; s.sq[1] = f[9]; s.sq[2] = (unsigned long long)nact; s.sq[3] = f[10];
            if (lead) { s.c_steps += 1; s.c_feas += (unsigned long long)nf; }
          }
        }
        if (lead) facc_reset(facc + 16 * ((t + 1) & 1), c.tid);  // read by everyone at the last attempt
        __syncthreads();
        SEQC_T(12);
        ++t;
        if (s.nf == 0) {  // F empty: reject the request atomically (R20)
          if (lead) req_reject(c, RL, OL, r);
          rejected = true;
          break;
        }
        // a5T: closeness of this CTA's feasible servers, top-2 keys into its slot (the
        // parameters computed once per CTA)
        __shared__ TopsisP tps;
        if (c.warp == 0) {  // lane k < 4: criterion k's FP64 norm and scale in parallel (R12)
          const int k = c.lane & 3;
          const double N = sqrt((double)s.sq[k]);
          const double sdk = N > 0 ? o.wd[k] / N : 0.0;
          double sd[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) sd[q] = __shfl_sync(FULL, sdk, q);
          if (c.lane == 0) {
            for (int q = 0; q < 4; ++q) { tps.mx[q] = s.mx[q]; tps.mn[q] = s.mn[q]; }
            topsis_params_sd(tps, sd);
          }
        }
        __syncthreads();
        SEQC_T(13);
        const TopsisP tp = tps;
        {
          // the thread's top-2 in FP32 (rows re-read from the CTA's copy: no registers held
          // across the barrier): servers ascend with j, so a strict > keeps the lowest index
          // first and an equal score lands in s2 (a tie, decided in FP64 below)
          // argmax of the closeness = argmin of q = Ed+^2 / Ed-^2 (topsis_q32: one reciprocal
          // instead of two square roots and a division; the warp kernel's decision rule)
          const float INF = __int_as_float(0x7f800000);
          float q1 = INF, q2 = INF;
          int j1 = -1;
#pragma unroll
          for (int j = 0; j < SQ_J; ++j) {
            if (!((okb >> j) & 1u)) continue;
            const int* m = mir + j * SQC_T + c.tid;
            const float qv = topsis_q32(tp, m[0], m[SQC_M], m[2 * SQC_M], m[3 * SQC_M]);
            if (j1 < 0 || qv < q1) { q2 = j1 < 0 ? q2 : q1; q1 = qv; j1 = j; }
            else if (qv < q2) q2 = qv;
          }
          // as keys for a max-merge: (0x7F800001 - bits(q), ~index) for the best (smaller q,
          // then the lower index, ranks higher; q = +inf still > 0); the second's index never
          // matters, only that it ranks below any best of the same q and is nonzero (0 = none)
          const int u1 = blockIdx.x * SQC_T + c.tid + max(j1, 0) * gridDim.x * SQC_T;
          const bool has2 = __popc(okb) >= 2;
          const unsigned long long k1 =
              j1 >= 0 ? ((unsigned long long)(0x7F800001u - __float_as_uint(q1)) << 32) | (0xFFFFFFFFu - (unsigned)u1)
                      : 0ull;
          const unsigned long long k2 =
              has2 ? ((unsigned long long)(0x7F800001u - __float_as_uint(q2)) << 32) | 1ull : 0ull;
          SEQC_T(14);
          block_top2(c, k1, k2);
          if (c.tid == 0) { kx[2 * q] = s.key1; kx[2 * q + 1] = s.key2; }
        }
        SEQC_T(5);
        cl.sync();  // (2) every CTA's keys
        SEQC_T(6);
        if (c.warp == 0) {  // a7: argmax, lowest index on ties (R14); FP64 near-tie re-decision
          unsigned long long k1 = c.lane < C ? kx[2 * c.lane] : 0ull, k2 = c.lane < C ? kx[2 * c.lane + 1] : 0ull;
          warp_top2(k1, k2);  // order-free merge: every lane holds the cluster's top-2
          if (c.lane == 0) {  // R14: near tie (relative q window, as the warp kernel) -> FP64
            const unsigned m1 = 0x7F800001u - (unsigned)(k1 >> 32), m2 = 0x7F800001u - (unsigned)(k2 >> 32);
            const float q1 = __uint_as_float(m1), q2 = __uint_as_float(m2);
            s.best = (int)(0xFFFFFFFFu - (unsigned)(k1 & 0xFFFFFFFFull));
            s.amb = o.exact64 || (k2 != 0ull && (m2 == m1 || q2 - q1 <= kTopsisDeltaQ * q1));
            s.thr = o.exact64 ? __int_as_float(0x7f800000) : q1 * (1.0f + 2.0f * kTopsisDeltaQ);
          }
        }
        __syncthreads();
        if (s.amb) {
          double bv = -DBL_MAX;
          int bj = -1;
#pragma unroll
          for (int j = 0; j < SQ_J; ++j) {
            if (!((okb >> j) & 1u)) continue;
            const int u = blockIdx.x * SQC_T + c.tid + j * gridDim.x * SQC_T;
            const int* m = mir + j * SQC_T + c.tid;
            const int x0 = m[0], x1 = m[SQC_M], x2 = m[2 * SQC_M], x3 = m[3 * SQC_M];
            if (topsis_q32(tp, x0, x1, x2, x3) > s.thr) continue;
            const double rr = topsis64(tp, x0, x1, x2, x3);
            if (rr > bv || (rr == bv && u < bj)) { bv = rr; bj = u; }
          }
          block_argmax64(c, bv, bj);
          if (c.tid == 0) { kxv[q] = s.bestv; kxi[q] = s.best; }
          cl.sync();  // (2') every CTA's FP64 candidate
          if (c.tid == 0) {
            double v = -DBL_MAX;
            int j = -1;
            for (int i = 0; i < C; ++i)
              if (kxi[i] >= 0 && (j < 0 || kxv[i] > v || (kxv[i] == v && kxi[i] < j))) { v = kxv[i]; j = kxi[i]; }
            s.best = j;
            if (lead) s.c_fp64 += 1;
          }
          __syncthreads();
        }
        SEQC_T(7);
        if (lead) commit_cta(c, RL, r, p);  // a8 on the live state (R16-R18)
        SEQC_T(8);
        cl.sync();  // (3) the commit (or its undo) is visible; the leader's verdict over DSMEM
        SEQC_T(4);
        if (c.tid == 0 && !lead) {
          const Scratch* ls = cl.map_shared_rank(&s, 0);
          const int u = s.best;
          s.fail = ls->fail;
          s.minfab = ls->minfab;
          if (s.fail) {  // R18: the same exclusion as the leader's
            for (int i = 0; i < s.nflow; ++i) if (s.fv[i] == u) s.fexcl[i] = 1;
            c.special[u >> 5] |= 1u << (u & 31);
            c.spok[u >> 5] &= ~(1u << (u & 31));
          } else {
            s.pod_srv[p] = u;
          }
        }
        __syncthreads();
        if (!s.fail) break;
      }
    }
    SEQC_T(9);
    if (!rejected && lead) req_finish(c, RL, OL, r, true);  // a9: top-up (R19), outputs
    SEQC_T(9);
    cl.sync();  // (4) the request's top-up / rollback is visible before the next one reads the state
    SEQC_T(4);
    if (c.tid == 0 && !lead) s.minfab = cl.map_shared_rank(&s, 0)->minfab;
    __syncthreads();
  }
  if (lead) flush_stats(c, stats);
#ifdef NACS_SEQC_PROF
  if (lead && c.tid == 0) {
    printf("filter: pre %llu loads %llu | prologue: head %llu flows %llu\n", seqc_prof_[21], seqc_prof_[20],
           seqc_prof_[23], seqc_prof_[22]);
    printf("commit ns: server %llu widest %llu path %llu vpath %llu | prologue: flows+clear %llu fabric %llu fok %llu\n",
           seqc_prof_[15], seqc_prof_[16], seqc_prof_[17], seqc_prof_[8], seqc_prof_[18], seqc_prof_[19], seqc_prof_[2]);
    printf("seqc ns: copy %llu begin %llu prologue %llu filter[loop %llu reduce %llu] barriers %llu "
           "score[stats %llu params %llu loop %llu top2 %llu] merge %llu commit %llu finish %llu\n",
           seqc_prof_[0], seqc_prof_[1], seqc_prof_[2], seqc_prof_[10], seqc_prof_[3], seqc_prof_[4], seqc_prof_[12],
           seqc_prof_[13], seqc_prof_[14], seqc_prof_[5], seqc_prof_[6] + seqc_prof_[7], seqc_prof_[8], seqc_prof_[9]);
  }
#endif
  cl.sync();  // no CTA leaves while another may still read its shared memory
}

// ------------------------------------------------------- simulator kernel ---
// Departure of accepted request r on the live state (thread 0): the exact inverse of its
// commit and top-up; f_u of its servers re-derived (R22).  st_set keeps the AHP presorted
// orders informed (touched servers).
__device__ void release_request(Ctx& c, const ReqsDev& R, const OutDev& O, int r) {
  const Geo& g = c.g;
  const int n = g.n;
  const int c0 = R.coff[r], c1 = R.coff[r + 1], v0 = R.voff[r], v1 = R.voff[r + 1];
  c.s->log_n = 0;  // releases are never undone
  for (int i = c0; i < c1; ++i) {
    const int u = O.server[i];
    st_set(c, u, c.st[u] + O.cpu_a[i]);
    st_set(c, n + u, c.st[n + u] + O.ram_a[i]);
  }
  for (int e = v0; e < v1; ++e) {
    const int us = O.server[c0 + R.src[e]], ud = O.server[c0 + R.dst[e]];
    if (us == ud) continue;  // host bus
    const int bw = O.bw_a[e];
    st_set(c, 3 * n + us, c.st[3 * n + us] + bw);
    st_set(c, 3 * n + ud, c.st[3 * n + ud] + bw);
    int off[4];
    const int m = path_links(g, us, ud, O.path[e], off);
    for (int t = 0; t < m; ++t) st_set(c, off[t], c.st[off[t]] + bw);
  }
  for (int i = c0; i < c1; ++i) {
    const int u = O.server[i];
    const int a = (c.st[u] < g.cpu_cap || c.st[n + u] < g.ram_cap) ? 1 : 0;
    if (c.st[2 * n + u] != a) st_set(c, 2 * n + u, a);
  }
  c.s->log_n = 0;
}

// The whole discrete-event run (reading R28) in ONE launch: one CTA keeps the event loop,
// the queue and the running set on the device, and schedules every attempt with the
// sequential machinery (run_request, keep) on the live state — no host round trip per
// attempt.  Per tick: departures (start + duration == t, in acceptance order), arrivals (in
// `order`, ascending arrival then id), FIFO scan (head-of-line blocking if hol), counters.
template <int METHOD>
__global__ void __launch_bounds__(512) k_simulate(Geo g, Opt o, int* state, ReqsDev R, OutDev O, int2* ulog,
                                                   float* ahp_ws, double* w64, unsigned long long* stats, SimDev S,
                                                   int smem_state) {
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ Scratch s;
  __shared__ int qn, nq2, next, blocked, done, cnt_s, cnt_l;
  __shared__ long long n_att, n_acc;
  Ctx c;
  init_ctx(c, g, o, &s);
  size_t off = 0;
  c.maskw = reinterpret_cast<unsigned*>(dyn + off);
  off = align16(off + sizeof(unsigned) * c.nW);
  c.special = reinterpret_cast<unsigned*>(dyn + off);
  off = align16(off + sizeof(unsigned) * c.nW);
  c.f0w = reinterpret_cast<unsigned*>(dyn + off);
  off = align16(off + sizeof(unsigned) * c.nW);
  c.edgebad = reinterpret_cast<unsigned*>(dyn + off);
  off = align16(off + sizeof(unsigned) * c.nEW);
  int* sst = smem_state ? load_state_smem(c, dyn + off, state) : state;
  c.st = sst;
  c.cr = c.st;
  c.snap = sst;
  c.ulog = ulog;
  c.nfcap = g.n;
  if (METHOD == 0) ahp_carve(c, reinterpret_cast<unsigned char*>(ahp_ws), g.n);
  c.w64 = w64;
  for (int w = c.tid; w < c.nW; w += c.B) { c.maskw[w] = 0u; c.special[w] = 0u; }
  for (int w = c.tid; w < c.nEW; w += c.B) c.edgebad[w] = 0u;
  for (int r = c.tid; r < R.n; r += c.B) { S.start[r] = -1; S.attempts[r] = 0; }
  for (int i = c.tid; i < S.max_ticks; i += c.B) S.head[i] = -1;
  if (c.tid == 0) { qn = 0; next = 0; done = 0; n_att = 0; n_acc = 0; }
  __syncthreads();
  init_minfab(c);  // departures raise residuals: the bound stays a lower bound
  int* qa = S.qbuf;
  int* qb = S.qtmp;
  int t = 0;
  for (; t < S.max_ticks; ++t) {
    // (1) departures first: the requests accepted with start + duration == t, kept in a
    // per-tick bucket (a linked list through S.run) so that a tick touches only its own
    if (c.tid == 0) {
      for (int r = S.head[t]; r >= 0; r = S.run[r]) release_request(c, R, O, r);
    }
    __syncthreads();
    // the presorted orders learn the released servers (before the first request there is
    // no presort yet: the first req_begin sorts the current state)
    if (METHOD == 0 && s.presorted) ahp_presort_update(c);
    // (2) arrivals
    if (c.tid == 0) {
      while (next < R.n && S.arrival[S.order[next]] == t) qa[qn++] = S.order[next++];
      nq2 = 0;
      blocked = 0;
    }
    __syncthreads();
    // (3) FIFO scan of the queue against the live state
    const int nq = qn;
    for (int i = 0; i < nq; ++i) {
      const int r = qa[i];
      if (blocked) {
        if (c.tid == 0) qb[nq2++] = r;
        continue;
      }
      run_request<METHOD>(c, R, O, r, true);
      if (c.tid == 0) {
        S.attempts[r] += 1;
        n_att += 1;
        if (O.status[r] == 1) {
          S.start[r] = t;
          const int end = t + S.duration[r];
          if (end < S.max_ticks) {
            S.run[r] = S.head[end];
            S.head[end] = r;
          }
          n_acc += 1;
        } else {
          qb[nq2++] = r;
          if (S.hol) blocked = 1;
        }
      }
      __syncthreads();
    }
    // (4) counters: active servers |N^s'|, active links |E^s'|, queue length
    if (c.tid == 0) { cnt_s = 0; cnt_l = 0; }
    __syncthreads();
    int as = 0, al = 0;
    for (int u = c.tid; u < g.n; u += c.B) as += c.st[2 * g.n + u];
    for (int l = c.tid; l < g.L; l += c.B) al += c.st[3 * g.n + l] < g.link_cap ? 1 : 0;
    for (int o2 = 16; o2; o2 >>= 1) {
      as += __shfl_xor_sync(FULL, as, o2);
      al += __shfl_xor_sync(FULL, al, o2);
    }
    if (c.lane == 0) { atomicAdd(&cnt_s, as); atomicAdd(&cnt_l, al); }
    __syncthreads();
    if (c.tid == 0) {
      qn = nq2;
      S.ticks[3 * t] = cnt_s;
      S.ticks[3 * t + 1] = cnt_l;
      S.ticks[3 * t + 2] = qn;
      done = qn == 0 && next == R.n;
    }
    {  // the survivors (qb) are the queue of the next tick; every thread swaps its copy
      int* tmp = qa;
      qa = qb;
      qb = tmp;
    }
    __syncthreads();
    if (done) { ++t; break; }
  }
  if (c.tid == 0) {
    S.totals[0] = t;
    S.totals[1] = n_att;
    S.totals[2] = n_acc;
  }
  if (smem_state) store_state_smem(c, sst, state);
  flush_stats(c, stats);
}

template <int METHOD>
__global__ void __launch_bounds__(1024) k_rank(Geo g, Opt o, int* state, QueryDev q, float* ahp_ws, double* w64,
                                               unsigned long long* stats) {
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ Scratch s;
  Ctx c;
  init_ctx(c, g, o, &s);
  size_t off = 0;
  c.maskw = reinterpret_cast<unsigned*>(dyn + off);
  off = align16(off + sizeof(unsigned) * c.nW);
  c.special = reinterpret_cast<unsigned*>(dyn + off);
  off = align16(off + sizeof(unsigned) * c.nW);
  c.f0w = reinterpret_cast<unsigned*>(dyn + off);
  off = align16(off + sizeof(unsigned) * c.nW);
  c.edgebad = reinterpret_cast<unsigned*>(dyn + off);
  c.st = state;
  c.cr = q.crit ? q.crit : c.st;
  c.snap = state;
  c.nfcap = g.n;
  if (METHOD == 0) {
    ahp_carve(c, reinterpret_cast<unsigned char*>(ahp_ws), g.n);
    c.w64 = w64;
  }
  clear_bitmaps(c);
  if (c.tid == 0) {
    s.dc = q.dc;
    s.dr = q.dr;
    s.nflow = q.nflow;
    int sumD = 0;
    for (int f = 0; f < q.nflow; ++f) { s.fv[f] = q.fv[f]; s.fD[f] = q.fD[f]; sumD += q.fD[f]; }
    s.sumD = sumD;
  }
  __syncthreads();
  if (o.path_filter && s.nflow > 0) fabric_tables(c);
  flow_server_ok(c);
  __syncthreads();
  // excluded servers (R18)
  for (int i = c.tid; i < q.nex; i += c.B) {
    int u = q.ex[i];
    atomicOr(&c.special[u >> 5], 1u << (u & 31));
    for (int f = 0; f < s.nflow; ++f)
      if (s.fv[f] == u) s.fexcl[f] = 1;
  }
  __syncthreads();
  bool wm = q.mask != nullptr && q.scores != nullptr;
  if (wm) pass_filter<true>(c, q.mask, q.scores);
  else pass_filter<false>(c, nullptr, nullptr);
  if (c.tid == 0) s.c_steps += 1;
  if (s.nf == 0) {
    if (c.tid == 0) *q.best = -1;
  } else {
    if (METHOD == 1) {
      if (wm) select_topsis<true>(c, q.scores);
      else select_topsis<false>(c, nullptr);
    } else {
      ahp_presort(c);
      if (wm) select_ahp<true>(c, q.scores);
      else select_ahp<false>(c, nullptr);
    }
    if (c.tid == 0) *q.best = s.best;
  }
  flush_stats(c, stats);
}

__global__ void k_validate(ReqsDev R, int* status, unsigned long long* stats) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R.n) return;
  int c0 = R.coff[r], v0 = R.voff[r];
  int bad = validate_request(R.coff[r + 1] - c0, R.voff[r + 1] - v0, R.cpu_min + c0, R.cpu_max + c0,
                             R.ram_min + c0, R.ram_max + c0, R.pod_of + c0, R.src + v0, R.dst + v0,
                             R.bw_min + v0, R.bw_max + v0);
  status[r] = bad ? -1 : 0;
  if (bad) atomicAdd(&stats[ST_INVALID], 1ull);
}

// ------------------------------------------------------ server sharding -----
// Sequential scheduling of one huge topology over G ranks (§8(e), C5): the state is
// replicated on every rank; per pod step each rank filters and reduces the statistics
// over all servers (replicated, exact), scores its own server block, and the ranks
// exchange their top-2 keys (ncclAllGather, 16 B per rank); every rank then takes the
// same decision and applies the same commit, so no state is ever exchanged.  The host
// drives the pod steps (nacs_api.cu, schedule_sharded); `ctl` tells it what comes next.
// Scratch lives in global memory because a request spans many launches.
enum { PH_DONE = 0, PH_NEWPOD = 1, PH_RETRY = 2, PH_FP64 = 3 };

__device__ void sh_ctx(Ctx& c, const Geo& g, const Opt& o, int* state, const ShardDev& d) {
  ctx_basic(c, g, o, d.gs);
  c.st = state;
  c.cr = c.st;
  c.snap = state;
  c.maskw = d.maskw;
  c.special = d.special;
  c.f0w = nullptr;  // R25 is not available on the sharded engine
  c.edgebad = d.edgebad;
  c.ulog = d.ulog;
  c.nfcap = g.n;
  if (o.method == 0 && d.ahp_ws) ahp_carve(c, d.ahp_ws, g.n);
}

// point the per-criterion level arrays of c at criterion k's slices
__device__ void ahp_slice(Ctx& c, const ShardDev& d, int k) {
  const int n2 = next_pow2(c.g.n);
  c.lvm = d.lvmC + (size_t)k * n2;
  c.lvw = d.lvwC + (size_t)k * n2;
  c.pa = d.paC + (size_t)k * (n2 + 2);
  c.pb = d.pbC + (size_t)k * (n2 + 2);
  c.lvl = d.lvlC + (size_t)k * c.g.n;
}

__device__ void sh_flush(Ctx& c, unsigned long long* stats) {
  flush_stats(c, stats);
  if (c.tid == 0) {
    Scratch* s = c.s;
    s->c_steps = s->c_retries = s->c_fp64 = s->c_invalid = s->c_feas = s->c_pairs = 0;
  }
}

template <int METHOD>
__global__ void __launch_bounds__(1024) k_sh_begin(Geo g, Opt o, int* state, ReqsDev R, OutDev O, int r,
                                                   ShardDev d, int first) {
  Ctx c;
  sh_ctx(c, g, o, state, d);
  Scratch* s = c.s;
  if (r == 0) init_minfab(c);  // the call's first request: the bound of the live state
  if (first == 2 && d.facc[15]) {  // AHP: k_presort_runs / _merge have just rebuilt the presorted orders
    for (int w = c.tid; w < c.nW; w += c.B) c.dirty[w] = 0u;
    if (c.tid == 0) { s->ntouched = 0; s->touch_over = 0; s->presorted = 1; }
    __syncthreads();
  }
  if (c.tid == 0) {
    s->c_steps = s->c_retries = s->c_fp64 = s->c_invalid = s->c_feas = s->c_pairs = 0;
    if (first == 1) { s->presorted = 0; s->touch_over = 0; s->ntouched = 0; }
    if (METHOD == 0) {
      double L1[4];
      ahp_l1_dev(o, L1);
      for (int k = 0; k < 4; ++k) { s->L1d[k] = L1[k]; s->L1[k] = (float)L1[k]; }
    }
  }
  __syncthreads();
  req_begin<METHOD>(c, R, r, true);
  if (!s->req_ok) {
    write_rejected(c, R, O, r, -1);
    __syncthreads();
    sh_flush(c, d.stats);
    if (c.tid == 0) d.ctl[0] = PH_DONE;
    return;
  }
  if (c.tid == 0) { d.ctl[0] = PH_NEWPOD; d.ctl[1] = 0; }
}

// AHP on the sharded engine: the presorted orders of the three criteria, rebuilt when the
// request is the call's first or the previous request overflowed the merge list (the
// decision is published in facc[15] for k_sh_begin, which resets the flags), from sorted
// runs: k_presort_runs sorts runs of SQP_RUN keys
// (value << 32 | server: unique, so every order is total) in shared memory, one CTA per run
// and criterion; k_presort_merge puts each key at its final position — its position in its
// run plus the count of smaller keys in every other run (binary searches).  (A bitonic sort
// over global memory by one CTA per criterion took 5 ms at C5.)
constexpr int SQP_RUN = 8192;  // keys per run (64 KB of shared memory)
__device__ __forceinline__ unsigned long long* presort_runs(const ShardDev& d, int ci, int P2) {
  const size_t off = ((size_t)ci * 5 * (P2 + 1) + 1) & ~(size_t)1;  // 8-byte aligned in the slice
  return reinterpret_cast<unsigned long long*>(d.lvscr + off);
}
__device__ __forceinline__ bool presort_needed(const ShardDev& d, int first) {
  const Scratch* gs = d.gs;
  return first || gs->touch_over || !gs->presorted;
}
__global__ void __launch_bounds__(1024) k_presort_runs(Geo g, int* state, ShardDev d, int first) {
  const bool need = presort_needed(d, first);
  if (blockIdx.x == 0 && threadIdx.x == 0) d.facc[15] = need ? 1ull : 0ull;
  if (!need) return;
  extern __shared__ unsigned long long sk[];
  const int n = g.n, P2 = next_pow2(n), S = min(P2, SQP_RUN), R = P2 / S;
  const int ci = blockIdx.x / R, run = blockIdx.x % R;
  const int* x = state + crit_of(ci) * n;
  for (int i = threadIdx.x; i < S; i += blockDim.x) {
    const int u = run * S + i;
    sk[i] = u < n ? ((unsigned long long)(unsigned)x[u] << 32) | (unsigned)u : ~0ull;
  }
  __syncthreads();
  for (int k = 2; k <= S; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < S; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const unsigned long long a = sk[i], b = sk[ixj];
          if ((a > b) == ((i & k) == 0)) { sk[i] = b; sk[ixj] = a; }
        }
      }
      __syncthreads();
    }
  }
  unsigned long long* out = presort_runs(d, ci, P2) + (size_t)run * S;
  for (int i = threadIdx.x; i < S; i += blockDim.x) out[i] = sk[i];
}
__global__ void __launch_bounds__(256) k_presort_merge(Geo g, ShardDev d, int first) {
  if (!presort_needed(d, first)) return;
  const int n = g.n, P2 = next_pow2(n), S = min(P2, SQP_RUN), R = P2 / S;
  unsigned short* perm = reinterpret_cast<unsigned short*>(d.ahp_ws);  // ahp_carve: perm first
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < 3 * P2; t += gridDim.x * blockDim.x) {
    const int ci = t / P2, i = t - ci * P2, run = i / S;
    const unsigned long long* runs = presort_runs(d, ci, P2);
    const unsigned long long key = runs[i];
    const int u = (int)(unsigned)(key & 0xffffffffull);
    if (key == ~0ull || u >= n) continue;
    int pos = i - run * S;
    for (int r2 = 0; r2 < R; ++r2) {
      if (r2 == run) continue;
      const unsigned long long* a = runs + (size_t)r2 * S;
      int lo = 0, hi = S;  // keys of run r2 below key
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (a[mid] < key) lo = mid + 1;
        else hi = mid;
      }
      pos += lo;
    }
    NACS_DCHECK(pos >= 0 && pos < n);
    perm[ci * P2 + pos] = (unsigned short)u;
  }
}

// pod prologue (new pod) + filter and statistics over all servers (replicated)
// The pod step's preparation in three launches: prep_a (1 CTA: flows, fabric tables,
// flow-server feasibility), k_sh_filter (the whole grid: filter and statistics over the
// 65536 servers of C5), prep_b (1 CTA: rejection, AHP levels and prefix sums).  The filter
// used to run in the one CTA of prep_a and was the largest item of a C5 pod step.
template <int METHOD>
__global__ void __launch_bounds__(1024) k_sh_prep_a(Geo g, Opt o, int* state, ReqsDev R, OutDev O, int r,
                                                    ShardDev d) {
  const int phase = d.ctl[0];
  if (phase != PH_NEWPOD && phase != PH_RETRY) return;
  Ctx c;
  sh_ctx(c, g, o, state, d);
  if (phase == PH_NEWPOD) pod_prologue(c, R, r, d.ctl[1]);
  if (c.tid < 11) d.facc[c.tid] = (c.tid >= 2 && c.tid <= 7 && !(c.tid & 1)) ? ~0ull : 0ull;
}

template <int METHOD>
__global__ void __launch_bounds__(1024) k_sh_filter(Geo g, Opt o, int* state, ShardDev d) {
  const int phase = d.ctl[0];
  if (phase != PH_NEWPOD && phase != PH_RETRY) return;
  Ctx c;
  sh_ctx(c, g, o, state, d);
  pass_filter<false, true>(c, nullptr, nullptr, d.facc);
}

// The grid filter's statistics (k_sh_filter, in facc) into the scratch fields, and for AHP
// each criterion's scale 9 / (max - min) (one thread).  count: the call's counters too.
__device__ void sh_prep_fields(Scratch* s, const unsigned long long* f, bool ahp, bool count) {
  const int nf = (int)f[0], nact = (int)f[1];
  s->nf = nf;
  s->nact = nact;
  s->mn[0] = (int)f[2]; s->mx[0] = (int)f[3];
  s->mn[1] = (int)f[4]; s->mx[1] = (int)f[5];
  s->mn[2] = nact == nf ? 1 : 0; s->mx[2] = nact > 0 ? 1 : 0;  // f_u in {0,1}
  s->mn[3] = (int)f[6]; s->mx[3] = (int)f[7];
  s->sq[0] = f[8]; s->sq[1] = f[9]; s->sq[2] = (unsigned long long)nact; s->sq[3] = f[10];
  if (count) {
    s->c_feas += (unsigned long long)nf;
    s->c_steps += 1;
  }
  if (ahp && nf > 0) {  // levels and pass-1 prefix sums of every non-constant criterion
    for (int k = 0; k < 4; ++k) {
      const int lo = s->mn[k], hi = s->mx[k];
      s->ahp_const[k] = hi == lo;
      const double sc = hi > lo ? 9.0 / (double)(hi - lo) : 0.0;
      s->ahp_scaled[k] = sc;
      s->ahp_scale[k] = (float)sc;
    }
  }
}

template <int METHOD>
__global__ void __launch_bounds__(1024) k_sh_prep(Geo g, Opt o, int* state, ReqsDev R, OutDev O, int r,
                                                  ShardDev d) {
  const int phase = d.ctl[0];
  if (phase != PH_NEWPOD && phase != PH_RETRY) return;
  Ctx c;
  sh_ctx(c, g, o, state, d);
  Scratch* s = c.s;
  if (c.tid == 0) sh_prep_fields(s, d.facc, METHOD == 0, true);
  __syncthreads();
  if (s->nf == 0) {
    req_reject(c, R, O, r);
    sh_flush(c, d.stats);
    if (c.tid == 0) d.ctl[0] = PH_DONE;
    return;
  }
}

// The AHP levels and pass-1 prefix sums of each non-constant criterion, one CTA per criterion
// (the three numeric criteria are independent; they ran one after another in k_sh_prep's one
// CTA).  Each CTA works on a shared-memory copy of the scratch block (its merge lists), its
// own slice of the sorting buffers (d.lvscr) and shared-memory copies of the feasibility and
// dirty bitmaps (the presorted walk looks both up at random servers).
__global__ void __launch_bounds__(1024) k_sh_levels(Geo g, Opt o, int* state, ShardDev d) {
  const int phase = d.ctl[0];
  if (phase != PH_NEWPOD && phase != PH_RETRY) return;
  const int k = blockIdx.x;
  const Scratch* gs = d.gs;
  if (gs->nf == 0) return;  // rejected in k_sh_prep
  const int n2 = next_pow2(g.n);
  if (gs->touch_over) {
    // the request touched more servers than the merge list holds: the presorted orders are
    // rebuilt (ahp_levels_of), which writes the shared orders and scratch — one CTA, in turn
    if (k != 0) return;
    Ctx c;
    sh_ctx(c, g, o, state, d);
    for (int kk = 0; kk < 4; ++kk) {
      if (c.s->ahp_const[kk]) {
        if (c.tid == 0) d.Kc[kk] = 0;
        continue;
      }
      ahp_slice(c, d, kk);
      const int K = ahp_levels_of(c, kk);
      ahp_prefix(c, K, c.lvm);
      for (int l = c.tid; l < K; l += c.B) { d.wq[kk * n2 + l] = 0.f; d.l2q[kk * n2 + l] = 0.f; }
      if (c.tid == 0) {
        d.Kc[kk] = K;
        c.s->c_pairs += (unsigned long long)K * (unsigned long long)(K - 1) / 2;
      }
      __syncthreads();
    }
    return;
  }
  if (gs->ahp_const[k]) {
    if (threadIdx.x == 0) d.Kc[k] = 0;
    return;
  }
  __shared__ Scratch ls;
  extern __shared__ unsigned sh_bits[];
  {  // the scratch block into shared memory (read-only here except the merge lists)
    const int* src = reinterpret_cast<const int*>(gs);
    int* dst = reinterpret_cast<int*>(&ls);
    for (int i = threadIdx.x; i < (int)(sizeof(Scratch) / 4); i += blockDim.x) dst[i] = src[i];
  }
  Ctx c;
  sh_ctx(c, g, o, state, d);
  c.s = &ls;
  for (int w = c.tid; w < c.nW; w += c.B) {
    sh_bits[w] = c.maskw[w];
    sh_bits[c.nW + w] = c.dirty[w];
  }
  __syncthreads();
  c.maskw = sh_bits;
  c.dirty = sh_bits + c.nW;
  int* sc = d.lvscr + (size_t)k * 5 * (n2 + 1);
  c.keys = reinterpret_cast<float*>(sc);
  c.sidx = sc + (n2 + 1);
  c.keys2 = reinterpret_cast<float*>(sc + 2 * (n2 + 1));
  c.sidx2 = sc + 3 * (n2 + 1);
  c.lst = sc + 4 * (n2 + 1);
  ahp_slice(c, d, k);
  const int K = ahp_levels_of(c, k);
  ahp_prefix(c, K, c.lvm);
  for (int l = c.tid; l < K; l += c.B) { d.wq[k * n2 + l] = 0.f; d.l2q[k * n2 + l] = 0.f; }
  if (c.tid == 0) {
    d.Kc[k] = K;
    atomicAdd(&d.gs->c_pairs, (unsigned long long)K * (unsigned long long)(K - 1) / 2);
  }
}

// ---- the same level extraction on a cluster of CL CTAs per criterion (k_sh_levels_cl) ----
// Every loop of presorted_collect / ahp_levels_sorted / ahp_prefix runs over the cluster's
// warps (global warp segments); the scans between warps become a CTA scan plus a scan over
// the CTAs' totals read over DSMEM; the work arrays (keys, levels, prefix sums) are the
// criterion's global slices as before.  The thread-0 merge list of touched servers is
// replicated in every CTA (each reads the same global values).  Same results as the one-CTA
// kernel: the same sorted order, levels and (exact, integer-valued) FP64 prefix sums.
struct ClSeg {
  int r, C;  // this CTA's rank in the cluster, cluster size
  int par;   // scan call parity
};
__device__ __forceinline__ void cl_seg(const Ctx& c, const ClSeg& q, int N, int& s0, int& s1) {
  const int GW = q.C * c.NW;
  const int seg = ((N + GW - 1) / GW + 31) & ~31;
  s0 = min((q.r * c.NW + c.warp) * seg, N);
  s1 = min(s0 + seg, N);
}
// exclusive scan over all warps of the cluster of one int per warp; *total = the sum
__device__ int cl_exscan(Ctx& c, ClSeg& q, cgx::cluster_group& cl, int x, int* total) {
  Scratch* s = c.s;
  int cta_total;
  const int r = warp_exscan(c, x, &cta_total);
  const int par = q.par;
  q.par ^= 1;
  if (c.tid == 0) s->cl_pub[par] = cta_total;
  cl.sync();
  if (c.warp == 0) {
    const int v = c.lane < q.C ? *cl.map_shared_rank(&s->cl_pub[par], c.lane) : 0;
    int iv = v;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(FULL, iv, o);
      if (c.lane >= o) iv += y;
    }
    const int base = __shfl_sync(FULL, iv - v, q.r), tot = __shfl_sync(FULL, iv, 31);
    if (c.lane == 0) { s->cl_base = base; s->cl_total = tot; }
  }
  __syncthreads();
  *total = s->cl_total;
  const int b = s->cl_base;
  __syncthreads();
  return r + b;
}
__device__ void cl_exscan_d2(Ctx& c, ClSeg& q, cgx::cluster_group& cl, double& a, double& b, double* ta, double* tb) {
  Scratch* s = c.s;
  double A, B;
  warp_exscan_d2(c, a, b, &A, &B);
  const int par = q.par;
  q.par ^= 1;
  if (c.tid == 0) { s->cl_pubd[par][0] = A; s->cl_pubd[par][1] = B; }
  cl.sync();
  if (c.warp == 0) {
    double va = 0.0, vb = 0.0;
    if (c.lane < q.C) {
      const double* rp = cl.map_shared_rank(&s->cl_pubd[par][0], c.lane);
      va = rp[0];
      vb = rp[1];
    }
    double ia = va, ib = vb;
    for (int o = 1; o < 32; o <<= 1) {
      const double ya = __shfl_up_sync(FULL, ia, o), yb = __shfl_up_sync(FULL, ib, o);
      if (c.lane >= o) { ia += ya; ib += yb; }
    }
    const double ba = __shfl_sync(FULL, ia - va, q.r), bb = __shfl_sync(FULL, ib - vb, q.r);
    const double sa = __shfl_sync(FULL, ia, 31), sb = __shfl_sync(FULL, ib, 31);
    if (c.lane == 0) { s->cl_based[0] = ba; s->cl_based[1] = bb; s->cl_totald[0] = sa; s->cl_totald[1] = sb; }
  }
  __syncthreads();
  a += s->cl_based[0];
  b += s->cl_based[1];
  *ta = s->cl_totald[0];
  *tb = s->cl_totald[1];
  __syncthreads();
}

// presorted_collect(c, ci, FEAS) over the cluster
template <bool FEAS>
__device__ int cl_collect(Ctx& c, ClSeg& q, cgx::cluster_group& cl, int ci) {
  Scratch* s = c.s;
  const int n = c.g.n, P2 = next_pow2(n);
  const int* x = c.cr + crit_of(ci) * n;
  const unsigned short* perm = c.perm + ci * P2;
  int s0, s1;
  cl_seg(c, q, n, s0, s1);
  int cnt = 0;
#pragma unroll 4
  for (int base = s0; base < s1; base += 32) {
    const int i = base + c.lane;
    const int u = i < s1 ? perm[i] : 0;
    const bool k = i < s1 && (!FEAS || feas_bit(c, u)) && !((c.dirty[u >> 5] >> (u & 31)) & 1u);
    cnt += __popc(__ballot_sync(FULL, k));
  }
  int mtot;
  int pos = cl_exscan(c, q, cl, cnt, &mtot);
#pragma unroll 4
  for (int base = s0; base < s1; base += 32) {
    const int i = base + c.lane;
    const int u = i < s1 ? perm[i] : 0;
    const bool k = i < s1 && (!FEAS || feas_bit(c, u)) && !((c.dirty[u >> 5] >> (u & 31)) & 1u);
    const unsigned bal = __ballot_sync(FULL, k);
    if (k) {
      const int qq = pos + __popc(bal & ((1u << c.lane) - 1u));
      NACS_DCHECK(qq >= 0 && qq < n);
      c.keys2[qq] = (float)x[u];
      c.sidx2[qq] = u;
    }
    pos += __popc(bal);
  }
  if (c.warp == 0) {  // touched (feasible) servers sorted by current value, ties in touch order
    // (the insertion sort of presorted_collect): warp 0 loads them at once, keeps the feasible
    // ones in order, and places each at its rank (every CTA)
    __shared__ float tv[2 * MAXC];
    __shared__ int tu[2 * MAXC];
    const int nt = min(s->ntouched, 2 * MAXC);
    int d = 0;
    for (int t0 = 0; t0 < nt; t0 += 32) {
      const int t = t0 + c.lane;
      const int u = t < nt ? s->touched[t] : 0;
      const bool keep = t < nt && (!FEAS || feas_bit(c, u));
      const float v = keep ? (float)x[u] : 0.f;
      const unsigned bal = __ballot_sync(FULL, keep);
      if (keep) {
        const int at = d + __popc(bal & ((1u << c.lane) - 1u));
        tv[at] = v;
        tu[at] = u;
      }
      d += __popc(bal);
    }
    __syncwarp();
    for (int t = c.lane; t < d; t += 32) {
      const float v = tv[t];
      int r = 0;
      for (int j = 0; j < d; ++j) {
        const float w = tv[j];
        r += (w < v) || (w == v && j < t);
      }
      s->dval[r] = v;
      s->dsrv[r] = tu[t];
    }
    if (c.lane == 0) s->nd = d;
  }
  cl.sync();  // keys2 / sidx2 complete; nd in every CTA
  const int m1 = mtot, d = s->nd;
  const int gt = q.r * c.B + c.tid, gB = q.C * c.B;
  for (int i = gt; i < m1; i += gB) {
    const float v = c.keys2[i];
    int lo = 0, hi = d;
    while (lo < hi) { int mid = (lo + hi) >> 1; if (s->dval[mid] < v) lo = mid + 1; else hi = mid; }
    NACS_DCHECK(i + lo < n);
    c.keys[i + lo] = v;
    c.sidx[i + lo] = c.sidx2[i];
  }
  for (int j = gt; j < d; j += gB) {
    const float v = s->dval[j];
    int lo = 0, hi = m1;
    while (lo < hi) { int mid = (lo + hi) >> 1; if (c.keys2[mid] <= v) lo = mid + 1; else hi = mid; }
    c.keys[j + lo] = v;
    c.sidx[j + lo] = s->dsrv[j];
  }
  cl.sync();
  return m1 + d;
}

// ahp_levels_sorted over the cluster
__device__ int cl_levels_sorted(Ctx& c, ClSeg& q, cgx::cluster_group& cl, int m) {
  int s0, s1;
  cl_seg(c, q, m, s0, s1);
  int cnt = 0;
#pragma unroll 4
  for (int base = s0; base < s1; base += 32) {
    const int i = base + c.lane;
    const bool f = i < s1 && (i == 0 || c.keys[i] != c.keys[i - 1]);
    cnt += __popc(__ballot_sync(FULL, f));
  }
  int K;
  int l0 = cl_exscan(c, q, cl, cnt, &K);
#pragma unroll 2
  for (int base = s0; base < s1; base += 32) {
    const int i = base + c.lane;
    const bool in = i < s1;
    const bool f = in && (i == 0 || c.keys[i] != c.keys[i - 1]);
    const unsigned bal = __ballot_sync(FULL, f);
    const int qq = l0 + __popc(bal & (0xffffffffu >> (31 - c.lane))) - 1;
    NACS_DCHECK(!in || (qq >= 0 && qq < m && c.sidx[i] >= 0 && c.sidx[i] < c.g.n));
    if (f) {
      c.lvm[qq].x = c.keys[i];
      c.lst[qq] = i;
    }
    if (in) c.lvl[c.sidx[i]] = qq;
    l0 += __popc(bal);
  }
  cl.sync();
  const int gt = q.r * c.B + c.tid, gB = q.C * c.B;
  for (int l = gt; l < K; l += gB) c.lvm[l].y = (float)((l + 1 < K ? c.lst[l + 1] : m) - c.lst[l]);
  cl.sync();
  return K;
}

// ahp_levels_active over the cluster
__device__ int cl_levels_active(Ctx& c, ClSeg& q, cgx::cluster_group& cl) {
  Scratch* s = c.s;
  const int n = c.g.n;
  const int nf = s->nf, nact = s->nact;
  const int K = (nact > 0) + (nact < nf);
  const int gt = q.r * c.B + c.tid, gB = q.C * c.B;
  for (int u = gt; u < n; u += gB)
    if (feas_bit(c, u)) c.lvl[u] = c.st[2 * n + u] ? (nact < nf ? 1 : 0) : 0;
  if (q.r == 0 && c.tid == 0) {
    int l = 0;
    if (nact < nf) c.lvm[l++] = make_float2(0.0f, (float)(nf - nact));
    if (nact > 0) c.lvm[l++] = make_float2(1.0f, (float)nact);
  }
  cl.sync();
  return K;
}

// ahp_prefix over the cluster
__device__ void cl_prefix(Ctx& c, ClSeg& q, cgx::cluster_group& cl, int K, const float2* lv) {
  int s0, s1;
  cl_seg(c, q, K, s0, s1);
  double ta = 0, tb = 0;
  for (int base = s0; base < s1; base += 32) {
    const int i = base + c.lane;
    if (i < s1) { const float2 e = lv[i]; ta += (double)e.y; tb += (double)e.y * (double)e.x; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) { ta += __shfl_xor_sync(FULL, ta, o); tb += __shfl_xor_sync(FULL, tb, o); }
  double TA, TB;
  cl_exscan_d2(c, q, cl, ta, tb, &TA, &TB);
  double ra = ta, rb = tb;
  for (int base = s0; base < s1; base += 32) {
    const int i = base + c.lane;
    double a = 0, b = 0;
    if (i < s1) { const float2 e = lv[i]; a = (double)e.y; b = (double)e.y * (double)e.x; }
    double ia = a, ib = b;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double ya = __shfl_up_sync(FULL, ia, o), yb = __shfl_up_sync(FULL, ib, o);
      if (c.lane >= o) { ia += ya; ib += yb; }
    }
    if (i < s1) { c.pa[i] = ra + (ia - a); c.pb[i] = rb + (ib - b); }
    ra += __shfl_sync(FULL, ia, 31);
    rb += __shfl_sync(FULL, ib, 31);
  }
  if (q.r == 0 && c.tid == 0) { c.pa[K] = TA; c.pb[K] = TB; }
}

// k_sh_levels on a cluster per criterion: grid = 4 clusters of C CTAs (criterion = cluster id)
__global__ void __launch_bounds__(1024) k_sh_levels_cl(Geo g, Opt o, int* state, ReqsDev R, OutDev O, int r,
                                                      ShardDev d) {
  const int phase = d.ctl[0];
  if (phase != PH_NEWPOD && phase != PH_RETRY) return;
  cgx::cluster_group cl = cgx::this_cluster();
  ClSeg q;
  q.r = (int)cl.block_rank();
  q.C = (int)cl.num_blocks();
  q.par = 0;
  const int k = blockIdx.x / q.C;
  Scratch* gs = d.gs;
  const int nf = (int)d.facc[0];
  if (blockIdx.x == 0) {  // k_sh_prep's work in CTA 0: the scratch fields, an empty F rejected (R20)
    Ctx c0;
    sh_ctx(c0, g, o, state, d);
    if (threadIdx.x == 0) sh_prep_fields(gs, d.facc, true, true);
    __syncthreads();
    if (nf == 0) {
      req_reject(c0, R, O, r);
      sh_flush(c0, d.stats);
      if (threadIdx.x == 0) d.ctl[0] = PH_DONE;
      return;
    }
  }
  if (nf == 0) return;  // the same in every CTA
  const int n2 = next_pow2(g.n);
  if (gs->touch_over) {  // the presorted orders are rebuilt: k_sh_levels' one-CTA path, CTA 0
    if (blockIdx.x != 0) return;
    Ctx c;
    sh_ctx(c, g, o, state, d);
    for (int kk = 0; kk < 4; ++kk) {
      if (c.s->ahp_const[kk]) {
        if (c.tid == 0) d.Kc[kk] = 0;
        continue;
      }
      ahp_slice(c, d, kk);
      const int K = ahp_levels_of(c, kk);
      ahp_prefix(c, K, c.lvm);
      for (int l = c.tid; l < K; l += c.B) { d.wq[kk * n2 + l] = 0.f; d.l2q[kk * n2 + l] = 0.f; }
      if (c.tid == 0) {
        d.Kc[kk] = K;
        c.s->c_pairs += (unsigned long long)K * (unsigned long long)(K - 1) / 2;
      }
      __syncthreads();
    }
    return;
  }
  __shared__ Scratch ls;
  extern __shared__ unsigned sh_bits[];
  {  // (CTA 0 may be writing the statistics fields of gs: every CTA sets its own from facc)
    const int* src = reinterpret_cast<const int*>(gs);
    int* dst = reinterpret_cast<int*>(&ls);
    for (int i = threadIdx.x; i < (int)(sizeof(Scratch) / 4); i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) sh_prep_fields(&ls, d.facc, true, false);
  __syncthreads();
  if (ls.ahp_const[k]) {
    if (q.r == 0 && threadIdx.x == 0) d.Kc[k] = 0;
    cl.sync();  // (a cluster's CTAs leave together: the others may still be in their scans)
    return;
  }
  Ctx c;
  sh_ctx(c, g, o, state, d);
  c.s = &ls;
  for (int w = c.tid; w < c.nW; w += c.B) {
    sh_bits[w] = c.maskw[w];
    sh_bits[c.nW + w] = c.dirty[w];
  }
  __syncthreads();
  c.maskw = sh_bits;
  c.dirty = sh_bits + c.nW;
  int* sc = d.lvscr + (size_t)k * 5 * (n2 + 1);
  c.keys = reinterpret_cast<float*>(sc);
  c.sidx = sc + (n2 + 1);
  c.keys2 = reinterpret_cast<float*>(sc + 2 * (n2 + 1));
  c.sidx2 = sc + 3 * (n2 + 1);
  c.lst = sc + 4 * (n2 + 1);
  ahp_slice(c, d, k);
  const int K = k == 2 ? cl_levels_active(c, q, cl) : cl_levels_sorted(c, q, cl, cl_collect<true>(c, q, cl, k == 3 ? 2 : k));
  cl_prefix(c, q, cl, K, c.lvm);
  const int gt = q.r * c.B + c.tid, gB = q.C * c.B;
  for (int l = gt; l < K; l += gB) { d.wq[k * n2 + l] = 0.f; d.l2q[k * n2 + l] = 0.f; }
  if (q.r == 0 && c.tid == 0) {
    d.Kc[k] = K;
    atomicAdd(&d.gs->c_pairs, (unsigned long long)K * (unsigned long long)(K - 1) / 2);
  }
  cl.sync();  // no CTA leaves while another may still read its shared memory
}

// After an accepted request on the grid engine (facc[14], set by sh_commit_advance): the
// touched servers re-merged into the three presorted orders (ahp_presort_update), one
// cluster per order; k_presort_update_fin then forgets the touched servers.
__global__ void __launch_bounds__(1024) k_presort_update_cl(Geo g, Opt o, int* state, ShardDev d) {
  if (!d.facc[14]) return;
  cgx::cluster_group cl = cgx::this_cluster();
  ClSeg q;
  q.r = (int)cl.block_rank();
  q.C = (int)cl.num_blocks();
  q.par = 0;
  const int ci = blockIdx.x / q.C;
  const int n2 = next_pow2(g.n);
  __shared__ Scratch ls;
  extern __shared__ unsigned sh_bits[];
  {
    const int* src = reinterpret_cast<const int*>(d.gs);
    int* dst = reinterpret_cast<int*>(&ls);
    for (int i = threadIdx.x; i < (int)(sizeof(Scratch) / 4); i += blockDim.x) dst[i] = src[i];
  }
  Ctx c;
  sh_ctx(c, g, o, state, d);
  c.s = &ls;
  for (int w = c.tid; w < c.nW; w += c.B) sh_bits[w] = c.dirty[w];
  __syncthreads();
  unsigned short* perm = c.perm;
  c.dirty = sh_bits;
  int* sc = d.lvscr + (size_t)ci * 5 * (n2 + 1);
  c.keys = reinterpret_cast<float*>(sc);
  c.sidx = sc + (n2 + 1);
  c.keys2 = reinterpret_cast<float*>(sc + 2 * (n2 + 1));
  c.sidx2 = sc + 3 * (n2 + 1);
  const int m = cl_collect<false>(c, q, cl, ci);  // ends with a cluster barrier: sidx complete
  for (int i = q.r * c.B + c.tid; i < m; i += q.C * c.B) perm[ci * n2 + i] = (unsigned short)c.sidx[i];
  cl.sync();  // no CTA leaves while another may still read its shared memory
}
__global__ void __launch_bounds__(256) k_presort_update_fin(Geo g, ShardDev d) {
  if (!d.facc[14]) return;
  __syncthreads();
  if (threadIdx.x == 0) {  // ahp_clear_dirty on the global scratch
    Scratch* s = d.gs;
    unsigned* dirty = reinterpret_cast<unsigned*>(d.ahp_ws + align16(6 * (size_t)next_pow2(g.n)));  // ahp_carve
    const int nt = min(s->ntouched, 2 * MAXC);
    for (int i = 0; i < nt; ++i) {
      const int u = s->touched[i];
      dirty[u >> 5] &= ~(1u << (u & 31));
    }
    s->ntouched = 0;
    d.facc[14] = 0ull;
  }
}

// TOPSIS: closeness of this rank's servers [lo, hi); top-2 keys into slot
__global__ void __launch_bounds__(1024) k_sh_score(Geo g, Opt o, int* state, int lo, int hi, int slot,
                                                   ShardDev d) {
  Ctx c;
  sh_ctx(c, g, o, state, d);
  Scratch* s = c.s;
  const int phase = d.ctl[0];
  if (phase != PH_NEWPOD && phase != PH_RETRY) {
    if (c.tid == 0) { d.kx[2 * slot] = 0ull; d.kx[2 * slot + 1] = 0ull; }
    return;
  }
  const int n = g.n;
  TopsisP tp;
  for (int k = 0; k < 4; ++k) { tp.mx[k] = s->mx[k]; tp.mn[k] = s->mn[k]; }
  topsis_params(tp, o.wd, s->sq);
  unsigned long long k1 = 0, k2 = 0;
  const int* st = c.st;
  for (int base = lo - (lo & 31) + c.warp * 32; base < hi; base += c.B) {
    const int u = base + c.lane;
    if (u < lo || u >= hi) continue;
    if (!((c.maskw[u >> 5] >> (u & 31)) & 1u)) continue;
    const float rr = topsis32(tp, st[u], st[n + u], st[2 * n + u], st[3 * n + u]);
    top2_insert(k1, k2, score_key(rr, u));
  }
  block_top2(c, k1, k2);
  if (c.tid == 0) { d.kx[2 * slot] = s->key1; d.kx[2 * slot + 1] = s->key2; }
}

// commit the decided server (s->best) and advance the pod loop
template <int METHOD>
__device__ void sh_commit_advance(Ctx& c, const ReqsDev& R, const OutDev& O, int r, const ShardDev& d) {
  Scratch* s = c.s;
  const int p = d.ctl[1];
  commit_cta(c, R, r, p);  // the widest paths over the whole CTA, the words read in parallel
  __syncthreads();
  if (c.tid == 0) { d.ctl[2] = s->best; d.ctl[3] = s->fail; }
  if (s->fail) {
    if (c.tid == 0) d.ctl[0] = PH_RETRY;
    return;
  }
  if (p + 1 == s->P) {
    req_finish(c, R, O, r, true);
    if (METHOD == 0) {  // the presorted orders: k_presort_update_cl (after this kernel) on clusters
      __syncthreads();
      if (c.tid == 0) {
        if (s->touch_over) s->presorted = 0;  // more than the merge list holds: sort again next request
        else d.facc[14] = 1ull;
      }
    }
    sh_flush(c, d.stats);
    if (c.tid == 0) d.ctl[0] = PH_DONE;
  } else if (c.tid == 0) {
    d.ctl[0] = PH_NEWPOD;
    d.ctl[1] = p + 1;
  }
}

// TOPSIS decision from the gathered keys of all ranks (R14), then commit
__global__ void __launch_bounds__(1024) k_sh_decide(Geo g, Opt o, int* state, ReqsDev R, OutDev O, int r,
                                                    int world, ShardDev d) {
  const int phase = d.ctl[0];
  if (phase != PH_NEWPOD && phase != PH_RETRY) return;
  Ctx c;
  sh_ctx(c, g, o, state, d);
  Scratch* s = c.s;
  if (c.tid == 0) {
    unsigned long long k1 = 0, k2 = 0;
    for (int q = 0; q < world; ++q) top2_merge(k1, k2, d.kx[2 * q], d.kx[2 * q + 1]);
    const float s1 = __uint_as_float((unsigned)(k1 >> 32)), s2 = __uint_as_float((unsigned)(k2 >> 32));
    s->best = (int)(0xFFFFFFFFu - (unsigned)(k1 & 0xFFFFFFFFull));
    s->amb = o.exact64 || (k2 != 0ull && s1 - s2 <= kTopsisDelta);
    s->thr = o.exact64 ? -1.0f : s1 - 2.0f * kTopsisDelta;
    if (s->amb) d.ctl[0] = PH_FP64;
  }
  __syncthreads();
  if (s->amb) return;
  sh_commit_advance<1>(c, R, O, r, d);
}

// TOPSIS FP64 re-decision: exact closeness of this rank's candidates (r32 >= thr)
__global__ void __launch_bounds__(1024) k_sh_fp64(Geo g, Opt o, int* state, int lo, int hi, int slot,
                                                  ShardDev d) {
  Ctx c;
  sh_ctx(c, g, o, state, d);
  Scratch* s = c.s;
  const int n = g.n;
  TopsisP tp;
  for (int k = 0; k < 4; ++k) { tp.mx[k] = s->mx[k]; tp.mn[k] = s->mn[k]; }
  topsis_params(tp, o.wd, s->sq);
  const float thr = s->thr;
  const int* st = c.st;
  double bv = -DBL_MAX;
  int bj = -1;
  for (int base = lo - (lo & 31) + c.warp * 32; base < hi; base += c.B) {
    const int u = base + c.lane;
    if (u < lo || u >= hi) continue;
    if (!((c.maskw[u >> 5] >> (u & 31)) & 1u)) continue;
    const int x0 = st[u], x1 = st[n + u], x2 = st[2 * n + u], x3 = st[3 * n + u];
    if (topsis32(tp, x0, x1, x2, x3) < thr) continue;
    const double rr = topsis64(tp, x0, x1, x2, x3);
    if (rr > bv || (rr == bv && u < bj)) { bv = rr; bj = u; }
  }
  block_argmax64(c, bv, bj);
  if (c.tid == 0) { d.kxv[slot] = s->bestv; d.kxi[slot] = s->best; }
}

__global__ void __launch_bounds__(1024) k_sh_decide64(Geo g, Opt o, int* state, ReqsDev R, OutDev O, int r,
                                                      int world, ShardDev d) {
  if (d.ctl[0] != PH_FP64) return;
  Ctx c;
  sh_ctx(c, g, o, state, d);
  Scratch* s = c.s;
  if (c.tid == 0) {
    double bv = -DBL_MAX;
    int bj = -1;
    for (int q = 0; q < world; ++q) {
      const double v = d.kxv[q];
      const int j = d.kxi[q];
      if (j < 0) continue;
      if (bj < 0 || v > bv || (v == bv && j < bj)) { bv = v; bj = j; }
    }
    s->best = bj;
    s->c_fp64 += 1;
  }
  __syncthreads();
  sh_commit_advance<1>(c, R, O, r, d);
}

// ---- AHP over the grid and the ranks.  The pairs (t, K-1-t) of criterion k's levels are
// split into `world` equal shares; a thread takes one pair.  Pass 1 writes the weights
// w_l = m_l / colsum(l) of its levels, pass 2 their L2; every other entry stays 0 so
// that a sum-allreduce over the ranks assembles the full arrays.
__device__ __forceinline__ bool sh_live(const ShardDev& d, bool fp64) {
  const int ph = d.ctl[0];
  return fp64 ? ph == PH_FP64 : (ph == PH_NEWPOD || ph == PH_RETRY);
}

template <int PASS, bool FP64>
__global__ void __launch_bounds__(256) k_ahp_pass(Geo g, Opt o, int q0, int q1, int world, ShardDev d) {
  if (!sh_live(d, FP64)) return;
  const Scratch* s = d.gs;
  const int n2 = next_pow2(g.n);
  const int m = s->nf;
  const int rule = o.ahp_rule;
  const int lane = threadIdx.x & 31;
  int a[4], b[4], total = 0;
  for (int k = 0; k < 4; ++k) {
    const int K = d.Kc[k], half = (K + 1) >> 1;
    a[k] = (int)((long long)half * q0 / world);
    b[k] = (int)((long long)half * q1 / world);
    total += b[k] - a[k];
  }
  // one warp per level pair (t, K-1-t): lanes split the K-1 terms
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < total; i += nwarps) {
    int k = 0, t = i;
    while (t >= b[k] - a[k]) { t -= b[k] - a[k]; ++k; }
    t += a[k];
    const int K = d.Kc[k];
    const double sd = s->ahp_scaled[k];
    const float sc = (float)sd;
    const float2* lvm = d.lvmC + (size_t)k * n2;
    const float2* lvw = d.lvwC + (size_t)k * n2;
    const double* pa = d.paC + (size_t)k * (n2 + 2);
    const double* pb = d.pbC + (size_t)k * (n2 + 2);
    for (int side = 0; side < 2; ++side) {
      const int l = side ? K - 1 - t : t;
      if (side && l == t) break;
      if (PASS == 1) {
        const double vl = lvm[l].x, ml = lvm[l].y;
        double rec = 0;
        if (FP64) {
          for (int q = lane; q < l; q += 32) {
            const double dd = vl - (double)lvm[q].x;
            rec += (double)lvm[q].y / (rule ? 1.0 + sd * dd : dd);
          }
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) rec += __shfl_xor_sync(FULL, rec, off);
        } else {
          rec = rule ? rsum_warp<false, 1>(lvm, 0, l, lvm[l].x, sc, lane) : rsum_warp<false, 0>(lvm, 0, l, lvm[l].x, sc, lane);
        }
        if (lane == 0) {
          const double cgt = pa[K] - pa[l + 1];
          const double G = (pb[K] - pb[l + 1]) - cgt * vl;  // sum_{k>l} m_k (v_k - v_l), exact
          const double col = rule ? cgt + sd * G + ml + rec : sd * G + ml + rec / sd;
          if (FP64) d.wq64[k * n2 + l] = ml / col;
          else d.wq[k * n2 + l] = (float)(ml / col);
        }
      } else {
        const double vl = lvw[l].x;
        double rec = 0, wl;
        if (FP64) {
          wl = d.wq64[k * n2 + l];
          for (int q = l + 1 + lane; q < K; q += 32) {
            const double dd = (double)lvw[q].x - vl;
            rec += d.wq64[k * n2 + q] / (rule ? 1.0 + sd * dd : dd);
          }
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) rec += __shfl_xor_sync(FULL, rec, off);
        } else {
          wl = (double)lvw[l].y;
          rec = rule ? rsum_warp<true, 1>(lvw, l + 1, K, lvw[l].x, sc, lane) : rsum_warp<true, 0>(lvw, l + 1, K, lvw[l].x, sc, lane);
        }
        if (lane == 0) {
          const double lin = vl * pa[l] - pb[l];  // sum_{k<l} w_k (v_l - v_k)
          const double L = rule ? pa[l] + sd * lin + wl + rec : sd * lin + wl + rec / sd;
          if (FP64) d.l2q64[k * n2 + l] = L / (double)m;
          else d.l2q[k * n2 + l] = (float)(L / (double)m);
        }
      }
    }
  }
}

// FP32 passes, register-tiled: a warp takes P consecutive levels and walks the union of
// their term ranges once, each loaded (value, weight) feeding all P levels (the pair-per-warp
// loop above re-read the level array from L2 once per level: L2-bandwidth bound at C5).
// Terms sit at absolute positions k = base + lane (base a multiple of 32) in groups of 4
// sharing one reciprocal; terms outside a level's range enter as weight 0 over 1.  Each lane
// sums <= 32 terms per level in FP32 before the FP64 accumulation, so the error bound behind
// ahp_delta_rel (chunks of <= 32 terms, any order) holds unchanged.
// ABOVE = pass 2 (terms q in (l, K), d = v_q - v_l); else pass 1 (q in [0, l), d = v_l - v_q).
template <bool ABOVE, int RULE, int P>
__device__ __forceinline__ void rsum_tile(const float2* arr, int K, int l0, int np, float sc, int lane,
                                          double (&out)[P]) {
  float v[P];
#pragma unroll
  for (int p = 0; p < P; ++p) { v[p] = arr[l0 + (p < np ? p : 0)].x; out[p] = 0.0; }
  const int lmax = l0 + np - 1;
  int kb = ABOVE ? ((l0 + 1) & ~31) : 0;
  const int kend = ABOVE ? K : lmax;
  while (kb < kend) {
    float a[P];
#pragma unroll
    for (int p = 0; p < P; ++p) a[p] = 0.f;
    // a block of 8 chunks all inside every level's range: the same terms in the same order
    // without the per-chunk range tests (they were ~20% of the executed instructions)
    const bool block_full = ABOVE ? (kb > lmax && kb + 1024 <= K) : (kb + 1024 <= l0);
    if (block_full) {
      const float2* ap = arr + kb + lane;
#pragma unroll
      for (int j = 0; j < 8; ++j, ap += 128) {
        const float2 o0 = ap[0], o1 = ap[32], o2 = ap[64], o3 = ap[96];
#pragma unroll
        for (int p = 0; p < P; ++p) {
          float d0 = ABOVE ? o0.x - v[p] : v[p] - o0.x, d1 = ABOVE ? o1.x - v[p] : v[p] - o1.x;
          float d2 = ABOVE ? o2.x - v[p] : v[p] - o2.x, d3 = ABOVE ? o3.x - v[p] : v[p] - o3.x;
          if (RULE) {
            d0 = fmaf(sc, d0, 1.0f);
            d1 = fmaf(sc, d1, 1.0f);
            d2 = fmaf(sc, d2, 1.0f);
            d3 = fmaf(sc, d3, 1.0f);
          }
          const float p01 = d0 * d1, p23 = d2 * d3;
          const float n01 = fmaf(o0.y, d1, o1.y * d0), n23 = fmaf(o2.y, d3, o3.y * d2);
          a[p] = fmaf(fmaf(n01, p23, n23 * p01), rcp_approx(p01 * p23), a[p]);
        }
      }
      kb += 1024;
#pragma unroll
      for (int p = 0; p < P; ++p) out[p] += (double)a[p];
      continue;
    }
    for (int j = 0; j < 8 && kb < kend; ++j, kb += 128) {
      const int k = kb + lane;
      const bool full = ABOVE ? (kb > lmax && kb + 128 <= K) : (kb + 128 <= l0);
      if (full) {
        const float2 o0 = arr[k], o1 = arr[k + 32], o2 = arr[k + 64], o3 = arr[k + 96];
#pragma unroll
        for (int p = 0; p < P; ++p) {
          float d0 = ABOVE ? o0.x - v[p] : v[p] - o0.x, d1 = ABOVE ? o1.x - v[p] : v[p] - o1.x;
          float d2 = ABOVE ? o2.x - v[p] : v[p] - o2.x, d3 = ABOVE ? o3.x - v[p] : v[p] - o3.x;
          if (RULE) {
            d0 = fmaf(sc, d0, 1.0f);
            d1 = fmaf(sc, d1, 1.0f);
            d2 = fmaf(sc, d2, 1.0f);
            d3 = fmaf(sc, d3, 1.0f);
          }
          const float p01 = d0 * d1, p23 = d2 * d3;
          const float n01 = fmaf(o0.y, d1, o1.y * d0), n23 = fmaf(o2.y, d3, o3.y * d2);
          a[p] = fmaf(fmaf(n01, p23, n23 * p01), rcp_approx(p01 * p23), a[p]);
        }
      } else {
        float2 o[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) o[i] = k + 32 * i < K ? arr[k + 32 * i] : make_float2(0.f, 0.f);
#pragma unroll
        for (int p = 0; p < P; ++p) {
          float d[4], w[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int q = k + 32 * i;
            const bool in = ABOVE ? (q > l0 + p && q < K) : (q < l0 + p);
            float di = ABOVE ? o[i].x - v[p] : v[p] - o[i].x;
            if (RULE) di = fmaf(sc, di, 1.0f);
            d[i] = in ? di : 1.0f;
            w[i] = in ? o[i].y : 0.f;
          }
          const float p01 = d[0] * d[1], p23 = d[2] * d[3];
          const float n01 = fmaf(w[0], d[1], w[1] * d[0]), n23 = fmaf(w[2], d[3], w[3] * d[2]);
          a[p] = fmaf(fmaf(n01, p23, n23 * p01), rcp_approx(p01 * p23), a[p]);
        }
      }
    }
#pragma unroll
    for (int p = 0; p < P; ++p) out[p] += (double)a[p];
  }
#pragma unroll
  for (int p = 0; p < P; ++p)
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) out[p] += __shfl_xor_sync(FULL, out[p], off);
}

#ifndef NACS_AHP_TILE
#define NACS_AHP_TILE 4
#endif
#ifndef NACS_AHP_MINB  // CTAs per SM (the register budget): A/B at C5 (scripts/ab_c5_ahp.py,
#define NACS_AHP_MINB 5  // 128-thread CTAs): 4 -> 393.5, 5 -> 390.5, 6 -> 402, 7 -> 401, 8 -> 406 us per pod step
#endif
#ifndef NACS_AHP_BLOCK
#define NACS_AHP_BLOCK 128
#endif
constexpr int kAhpTile = NACS_AHP_TILE;

// The rank's pairs (t, K-1-t), t in [a, b), cut into tiles of kAhpTile consecutive t: a warp
// takes the low levels t.. and the mirrored high levels K-1-t.. of one tile (K-1 terms per
// pair, as before), skipping the middle level of an odd K on the high side.
template <int PASS, int RULE>
__global__ void __launch_bounds__(NACS_AHP_BLOCK, NACS_AHP_MINB) k_ahp_pass_tiled(Geo g, int q0, int q1, int world, ShardDev d) {
  constexpr int P = kAhpTile;
  if (!sh_live(d, false)) return;
  const Scratch* s = d.gs;
  const int n2 = next_pow2(g.n);
  const int m = s->nf;
  const int lane = threadIdx.x & 31;
  // ranks split whole tiles: tile starts are multiples of P for every world size, so the
  // FP32 chunking of each level's terms (rsum_tile, from l0) never depends on the split and
  // every rank count gives bit-identical weights and L2
  // the split and the criteria order once per CTA (thread 0: 64-bit divisions), then shared
  __shared__ int s_ab[2][4], s_ord[4], s_total;
  if (threadIdx.x == 0) {
    int total = 0;
    for (int k = 0; k < 4; ++k) {
      const int K = d.Kc[k], half = (K + 1) >> 1, ntile = (half + P - 1) / P;
      s_ab[0][k] = min(half, P * (int)((long long)ntile * q0 / world));
      s_ab[1][k] = min(half, P * (int)((long long)ntile * q1 / world));
      total += (s_ab[1][k] - s_ab[0][k] + P - 1) / P;
    }
    // criteria in decreasing K (a tile costs ~P (K-1) terms): the longest tiles start first
    int ord[4] = {0, 1, 2, 3};
    for (int x = 1; x < 4; ++x)
      for (int y = x; y > 0 && d.Kc[ord[y]] > d.Kc[ord[y - 1]]; --y) {
        const int tmp = ord[y]; ord[y] = ord[y - 1]; ord[y - 1] = tmp;
      }
    for (int k = 0; k < 4; ++k) s_ord[k] = ord[k];
    s_total = total;
  }
  __syncthreads();
  int a[4], b[4], ord[4];
  for (int k = 0; k < 4; ++k) { a[k] = s_ab[0][k]; b[k] = s_ab[1][k]; ord[k] = s_ord[k]; }
  const int total = s_total;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
#ifndef NACS_AHP_STATIC
  // tiles handed out in order (largest K first) from a counter: the warps that drew short
  // tiles take more, so the SMs run dry together; the last warp out resets the counters for
  // the next launch (facc[12] tiles, facc[13] warps done)
  unsigned long long* ctr = d.facc + 12;
  for (;;) {
    int i = 0;
    if (lane == 0) i = (int)atomicAdd(ctr, 1ull);
    i = __shfl_sync(FULL, i, 0);
    if (i >= total) {
      if (lane == 0 && atomicAdd(ctr + 1, 1ull) == (unsigned long long)(nwarps - 1)) {
        ctr[0] = 0ull;
        ctr[1] = 0ull;
      }
      break;
    }
#else
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < total; i += nwarps) {
#endif
    int j = 0, t = i;
    while (t >= (b[ord[j]] - a[ord[j]] + P - 1) / P) { t -= (b[ord[j]] - a[ord[j]] + P - 1) / P; ++j; }
    const int k = ord[j];
    const int K = d.Kc[k];
    const int t0 = a[k] + t * P, nt = min(P, b[k] - t0);
    const double sd = s->ahp_scaled[k];
    const float sc = (float)sd;
    const float2* lvm = d.lvmC + (size_t)k * n2;
    const float2* lvw = d.lvwC + (size_t)k * n2;
    const double* pa = d.paC + (size_t)k * (n2 + 2);
    const double* pb = d.pbC + (size_t)k * (n2 + 2);
    for (int side = 0; side < 2; ++side) {
      int l0 = side ? K - (t0 + nt) : t0, np = nt;
      if (side && l0 == t0 + nt - 1) { ++l0; --np; }  // the middle level, already on the low side
      if (np <= 0) continue;
      double rec[P];
      if (PASS == 1) rsum_tile<false, RULE, P>(lvm, K, l0, np, sc, lane, rec);
      else rsum_tile<true, RULE, P>(lvw, K, l0, np, sc, lane, rec);
#pragma unroll
      for (int p = 0; p < P; ++p) {
        if (lane != p || p >= np) continue;
        const int l = l0 + p;
        if (PASS == 1) {
          const double vl = lvm[l].x, ml = lvm[l].y;
          const double cgt = pa[K] - pa[l + 1];
          const double G = (pb[K] - pb[l + 1]) - cgt * vl;  // sum_{k>l} m_k (v_k - v_l), exact
          const double col = RULE ? cgt + sd * G + ml + rec[p] : sd * G + ml + rec[p] / sd;
          d.wq[k * n2 + l] = (float)(ml / col);
        } else {
          const double vl = lvw[l].x, wl = (double)lvw[l].y;
          const double lin = vl * pa[l] - pb[l];  // sum_{k<l} w_k (v_l - v_k)
          const double L = RULE ? pa[l] + sd * lin + wl + rec[p] : sd * lin + wl + rec[p] / sd;
          d.l2q[k * n2 + l] = (float)(L / (double)m);
        }
      }
    }
  }
}

// between the passes (1 CTA): (value, weight) levels and their prefix sums
template <bool FP64>
// one CTA per criterion (independent): the block scans of ahp_prefix run on a private
// shared-memory scratch block
__global__ void __launch_bounds__(1024) k_ahp_mid(Geo g, Opt o, int* state, ShardDev d) {
  if (!sh_live(d, FP64)) return;
  __shared__ Scratch ls;
  Ctx c;
  sh_ctx(c, g, o, state, d);
  c.s = &ls;
  const int n2 = next_pow2(g.n);
  {
    const int k = blockIdx.x;
    const int K = d.Kc[k];
    if (K == 0) return;
    ahp_slice(c, d, k);
    for (int l = c.tid; l < K; l += c.B)
      c.lvw[l] = make_float2(c.lvm[l].x, FP64 ? 0.f : d.wq[k * n2 + l]);
    __syncthreads();
    if (!FP64) {
      ahp_prefix(c, K, c.lvw);
    } else {  // exact prefix sums of the FP64 weights (serial in level order: rare path)
      if (c.tid == 0) {
        double a = 0, b = 0;
        for (int l = 0; l < K; ++l) {
          c.pa[l] = a;
          c.pb[l] = b;
          a += d.wq64[k * n2 + l];
          b += d.wq64[k * n2 + l] * (double)c.lvm[l].x;
        }
        c.pa[K] = a;
        c.pb[K] = b;
      }
      __syncthreads();
    }
  }
}

// k_ahp_mid in FP32 as two grid kernels.  ahp_prefix on a 1024-thread CTA cuts K into 32
// warp segments; these kernels run the same 32 segments, with the same loops, butterflies and
// shuffle scans (bit-identical prefix sums), as 8 CTAs of 4 warps per criterion instead of 32
// warps sharing one SM (ncu: the one-CTA version was issue-limited on that SM).
constexpr int kMidWarps = AHP_MID_WARPS;  // a multiple of 32
constexpr int kMidPer = kMidWarps / 32;     // segment totals per lane in k_ahp_mid_b's scan
__device__ __forceinline__ void mid_seg(int K, int w, int& s0, int& s1) {
  const int seg = ((K + kMidWarps - 1) / kMidWarps + 31) & ~31;
  s0 = min(w * seg, K);
  s1 = min(s0 + seg, K);
}

// (value, weight) levels of the segment and its totals
__global__ void __launch_bounds__(128) k_ahp_mid_a(Geo g, ShardDev d) {
  if (!sh_live(d, false)) return;
  const int k = blockIdx.y, K = d.Kc[k];
  if (K == 0) return;
  const int w = blockIdx.x * 4 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  const int n2 = next_pow2(g.n);
  const float2* lvm = d.lvmC + (size_t)k * n2;
  float2* lvw = d.lvwC + (size_t)k * n2;
  int s0, s1;
  mid_seg(K, w, s0, s1);
  double ta = 0, tb = 0;
  for (int base = s0; base < s1; base += 32) {
    const int i = base + lane;
    if (i < s1) {
      const float2 e = make_float2(lvm[i].x, d.wq[k * n2 + i]);
      lvw[i] = e;
      ta += (double)e.y;
      tb += (double)e.y * (double)e.x;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) { ta += __shfl_xor_sync(FULL, ta, o); tb += __shfl_xor_sync(FULL, tb, o); }
  if (lane == 0) {
    d.midtot[(k * kMidWarps + w) * 2] = ta;
    d.midtot[(k * kMidWarps + w) * 2 + 1] = tb;
  }
}

// exclusive scan of the segment totals (warp_exscan_d2's order), then the segment's prefixes
__global__ void __launch_bounds__(128) k_ahp_mid_b(Geo g, ShardDev d) {
  if (!sh_live(d, false)) return;
  const int k = blockIdx.y, K = d.Kc[k];
  if (K == 0) return;
  const int w = blockIdx.x * 4 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  const int n2 = next_pow2(g.n);
  const float2* lv = d.lvwC + (size_t)k * n2;
  double* pa = d.paC + (size_t)k * (n2 + 2);
  double* pb = d.pbC + (size_t)k * (n2 + 2);
  // lane L holds segments L*kMidPer ..: their exclusive prefixes within the lane, then a
  // warp scan of the lane sums
  double pa_l[kMidPer], pb_l[kMidPer], xa = 0.0, xb = 0.0;
#pragma unroll
  for (int j = 0; j < kMidPer; ++j) {
    pa_l[j] = xa;
    pb_l[j] = xb;
    xa += d.midtot[(k * kMidWarps + lane * kMidPer + j) * 2];
    xb += d.midtot[(k * kMidWarps + lane * kMidPer + j) * 2 + 1];
  }
  double ia = xa, ib = xb;
  for (int o = 1; o < 32; o <<= 1) {
    const double ya = __shfl_up_sync(FULL, ia, o), yb = __shfl_up_sync(FULL, ib, o);
    if (lane >= o) { ia += ya; ib += yb; }
  }
  double qa = pa_l[0], qb = pb_l[0];
#pragma unroll
  for (int j = 1; j < kMidPer; ++j)
    if (j == w % kMidPer) { qa = pa_l[j]; qb = pb_l[j]; }
  // segment w's exclusive prefix: its lane's exclusive prefix plus its offset in the lane
  double ra = __shfl_sync(FULL, ia - xa, w / kMidPer) + __shfl_sync(FULL, qa, w / kMidPer);
  double rb = __shfl_sync(FULL, ib - xb, w / kMidPer) + __shfl_sync(FULL, qb, w / kMidPer);
  const double TA = __shfl_sync(FULL, ia, 31), TB = __shfl_sync(FULL, ib, 31);
  int s0, s1;
  mid_seg(K, w, s0, s1);
  for (int base = s0; base < s1; base += 32) {
    const int i = base + lane;
    double a = 0, b = 0;
    if (i < s1) { const float2 e = lv[i]; a = (double)e.y; b = (double)e.y * (double)e.x; }
    double ja = a, jb = b;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double ya = __shfl_up_sync(FULL, ja, o), yb = __shfl_up_sync(FULL, jb, o);
      if (lane >= o) { ja += ya; jb += yb; }
    }
    if (i < s1) { pa[i] = ra + (ja - a); pb[i] = rb + (jb - b); }
    ra += __shfl_sync(FULL, ja, 31);
    rb += __shfl_sync(FULL, jb, 31);
  }
  if (w == 0 && lane == 0) { pa[K] = TA; pb[K] = TB; }
}

// k_ahp_mid_a + _b in one launch: a thread-block cluster per criterion (criterion = cluster
// id), the segment totals scanned over DSMEM (cl_exscan_d2) instead of through global memory
// between two kernels.  Same (value, weight) levels; the FP64 prefix sums in another order
// (segments of the cluster's warps).
__global__ void __launch_bounds__(1024) k_ahp_mid_cl(Geo g, ShardDev d) {
  if (!sh_live(d, false)) return;
  cgx::cluster_group cl = cgx::this_cluster();
  ClSeg q;
  q.r = (int)cl.block_rank();
  q.C = (int)cl.num_blocks();
  q.par = 0;
  const int k = blockIdx.x / q.C, K = d.Kc[k];
  if (K == 0) return;  // the same in every CTA of the cluster
  __shared__ Scratch ls;
  Ctx c;
  c.s = &ls;
  c.tid = threadIdx.x;
  c.B = blockDim.x;
  c.NW = blockDim.x >> 5;
  c.lane = threadIdx.x & 31;
  c.warp = threadIdx.x >> 5;
  const int n2 = next_pow2(g.n);
  const float2* lvm = d.lvmC + (size_t)k * n2;
  float2* lvw = d.lvwC + (size_t)k * n2;
  const float* wq = d.wq + (size_t)k * n2;
  double* pa = d.paC + (size_t)k * (n2 + 2);
  double* pb = d.pbC + (size_t)k * (n2 + 2);
  int s0, s1;
  cl_seg(c, q, K, s0, s1);
  double ta = 0, tb = 0;
  for (int base = s0; base < s1; base += 32) {
    const int i = base + c.lane;
    if (i < s1) {
      const float2 e = make_float2(lvm[i].x, wq[i]);
      lvw[i] = e;
      ta += (double)e.y;
      tb += (double)e.y * (double)e.x;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) { ta += __shfl_xor_sync(FULL, ta, o); tb += __shfl_xor_sync(FULL, tb, o); }
  double TA, TB;
  cl_exscan_d2(c, q, cl, ta, tb, &TA, &TB);  // ta, tb: this segment's exclusive prefix
  double ra = ta, rb = tb;
  for (int base = s0; base < s1; base += 32) {
    const int i = base + c.lane;
    double a = 0, b = 0;
    if (i < s1) { const float2 e = lvw[i]; a = (double)e.y; b = (double)e.y * (double)e.x; }
    double ja = a, jb = b;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double ya = __shfl_up_sync(FULL, ja, o), yb = __shfl_up_sync(FULL, jb, o);
      if (c.lane >= o) { ja += ya; jb += yb; }
    }
    if (i < s1) { pa[i] = ra + (ja - a); pb[i] = rb + (jb - b); }
    ra += __shfl_sync(FULL, ja, 31);
    rb += __shfl_sync(FULL, jb, 31);
  }
  if (q.r == 0 && c.tid == 0) { pa[K] = TA; pb[K] = TB; }
  cl.sync();  // no CTA leaves while another may still read its shared memory
}

// PG over F on the whole grid (FP32; one server per thread): each CTA leaves its top-2
// (score, index) keys in d.kpart for k_ahp_decide.  The top-2 of the union of per-CTA top-2
// sets is the global top-2, so the decision is the one-CTA kernel's.
template <bool FP64>
__device__ void ahp_decide_cta(const Geo& g, const Opt& o, int* state, const ReqsDev& R, const OutDev& O, int r,
                               const ShardDev& d);
__global__ void __launch_bounds__(1024) k_ahp_pg(Geo g, Opt o, int* state, ReqsDev R, OutDev O, int r,
                                                 ShardDev d) {
  if (!sh_live(d, false)) return;
  __shared__ Scratch ls;
  Ctx c;
  sh_ctx(c, g, o, state, d);
  const Scratch* gs = d.gs;
  c.s = &ls;
  const int n = g.n, n2 = next_pow2(n);
  const float inv_nf = rcp_approx((float)gs->nf);
  float L1[4];
  bool cst[4];
  for (int k = 0; k < 4; ++k) { L1[k] = gs->L1[k]; cst[k] = gs->ahp_const[k]; }
  unsigned long long k1 = 0, k2 = 0;
  for (int u = blockIdx.x * c.B + c.tid; u < n; u += gridDim.x * c.B) {
    if (!feas_bit(c, u)) continue;
    float pgv = 0.f;
    for (int k = 0; k < 4; ++k) {
      if (cst[k]) pgv += L1[k] * inv_nf;
      else pgv = fmaf(L1[k], d.l2q[k * n2 + d.lvlC[(size_t)k * n + u]], pgv);
    }
    top2_insert(k1, k2, score_key(pgv, u));
  }
  block_top2(c, k1, k2);
  // the last CTA to finish takes the decision (k_ahp_decide's FP32 path) in the same launch
  __shared__ bool last;
  if (c.tid == 0) {
    d.kpart[2 * blockIdx.x] = ls.key1;
    d.kpart[2 * blockIdx.x + 1] = ls.key2;
    __threadfence();
    last = atomicAdd(d.facc + 11, 1ull) == (unsigned long long)(gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  if (c.tid == 0) d.facc[11] = 0ull;  // for the next pod step
  __threadfence();
  ahp_decide_cta<false>(g, o, state, R, O, r, d);
}

// decide (1 CTA): PG over F, argmax (top-2 and near-tie test in FP32), commit
template <bool FP64>
__device__ void ahp_decide_cta(const Geo& g, const Opt& o, int* state, const ReqsDev& R, const OutDev& O, int r,
                               const ShardDev& d) {
  Ctx c;
  sh_ctx(c, g, o, state, d);
  Scratch* s = c.s;
  const int n = g.n, n2 = next_pow2(n), nf = s->nf;
  if (!FP64) {
    // the per-CTA top-2 keys of k_ahp_pg (PG over F on the whole grid), reduced here
    unsigned long long k1 = 0, k2 = 0;
    for (int i = c.tid; i < 2 * d.npart; i += c.B) top2_insert(k1, k2, __ldcg(d.kpart + i));
    block_top2(c, k1, k2);
    const float drel = ahp_delta_rel(nf);
    if (c.tid == 0) {
      const float s1 = __uint_as_float((unsigned)(s->key1 >> 32));
      const float s2 = __uint_as_float((unsigned)(s->key2 >> 32));
      s->best = (int)(0xFFFFFFFFu - (unsigned)(s->key1 & 0xFFFFFFFFull));
      s->amb = o.exact64 || (s->key2 != 0ull && s2 >= s1 * (1.0f - drel));
      if (s->amb) d.ctl[0] = PH_FP64;
    }
    __syncthreads();
    if (s->amb) {  // the FP64 passes start from zeroed weights and the pass-1 prefix sums
      for (int k = 0; k < 4; ++k) {
        const int K = d.Kc[k];
        if (K == 0) continue;
        for (int l = c.tid; l < K; l += c.B) { d.wq64[k * n2 + l] = 0.0; d.l2q64[k * n2 + l] = 0.0; }
        ahp_slice(c, d, k);
        ahp_prefix(c, K, c.lvm);
      }
      return;
    }
  } else {
    double bv = -DBL_MAX;
    int bj = -1;
    for (int u = c.tid; u < n; u += c.B) {
      if (!feas_bit(c, u)) continue;
      double v = 0;
      for (int k = 0; k < 4; ++k) {
        if (s->ahp_const[k]) v += s->L1d[k] / (double)nf;
        else v += s->L1d[k] * d.l2q64[k * n2 + d.lvlC[(size_t)k * n + u]];
      }
      if (v > bv || (v == bv && u < bj)) { bv = v; bj = u; }
    }
    block_argmax64(c, bv, bj);
    if (c.tid == 0) s->c_fp64 += 1;
  }
  sh_commit_advance<0>(c, R, O, r, d);
}
template <bool FP64>
__global__ void __launch_bounds__(1024) k_ahp_decide(Geo g, Opt o, int* state, ReqsDev R, OutDev O, int r,
                                                     ShardDev d) {
  if (!sh_live(d, FP64)) return;
  ahp_decide_cta<FP64>(g, o, state, R, O, r, d);
}

// CTAs per criterion of the sharded engine's AHP level extraction (1: k_sh_levels, one CTA)
static int sh_levels_cluster() {
  // A/B at C5 (scripts/ab_c5_ahp.py, 12 requests): 1 -> 645, 4 -> 518, 8 -> 492, 16 -> 479 us per pod step
  int C = 16;
  if (const char* e = getenv("NACS_LEVELS_CLUSTER")) C = atoi(e);  // experiments: 1, 2, 4, 8, 16
  return C < 1 || C > 16 ? 16 : C;
}

// CTAs per criterion of the between-passes kernel (1: k_ahp_mid_a / _b over 128 warps)
// (A/B at C5, 3 runs each: 1 -> 386.6, 16 -> 382.7 us per pod step, identical placements)
static int mid_cluster() {
  int C = 16;
  if (const char* e = getenv("NACS_MID_CLUSTER")) C = atoi(e);  // experiments: 1, 2, 4, 8, 16
  return C < 1 || C > 16 ? 16 : C;
}

cudaError_t launch_ahp_pass(int pass, bool fp64, const Geo& g, const Opt& o, int* state, int q0, int q1, int world,
                            const ShardDev& d, int num_sms, cudaStream_t st) {
  (void)state;
  const int blocks = num_sms * 8;
  if (!fp64) {
    // one resident wave of CTAs, the tiles from the counter (A/B: 387.3 vs 390.6 us per C5
    // pod step with 2368 CTAs)
    const int tb = num_sms * NACS_AHP_MINB;
    (void)blocks;
    if (pass == 1 && o.ahp_rule) k_ahp_pass_tiled<1, 1><<<tb, NACS_AHP_BLOCK, 0, st>>>(g, q0, q1, world, d);
    else if (pass == 1) k_ahp_pass_tiled<1, 0><<<tb, NACS_AHP_BLOCK, 0, st>>>(g, q0, q1, world, d);
    else if (o.ahp_rule) k_ahp_pass_tiled<2, 1><<<tb, NACS_AHP_BLOCK, 0, st>>>(g, q0, q1, world, d);
    else k_ahp_pass_tiled<2, 0><<<tb, NACS_AHP_BLOCK, 0, st>>>(g, q0, q1, world, d);
  } else if (pass == 1) {
    k_ahp_pass<1, true><<<blocks, 256, 0, st>>>(g, o, q0, q1, world, d);
  } else {
    k_ahp_pass<2, true><<<blocks, 256, 0, st>>>(g, o, q0, q1, world, d);
  }
  return cudaGetLastError();
}
cudaError_t launch_ahp_mid(bool fp64, const Geo& g, const Opt& o, int* state, const ShardDev& d, cudaStream_t st) {
  if (fp64) {
    k_ahp_mid<true><<<4, 1024, 0, st>>>(g, o, state, d);
  } else {
    const int CL = mid_cluster();
    if (CL <= 1) {
      k_ahp_mid_a<<<dim3(kMidWarps / 4, 4), 128, 0, st>>>(g, d);
      k_ahp_mid_b<<<dim3(kMidWarps / 4, 4), 128, 0, st>>>(g, d);
    } else {
      cudaError_t e;
      if (CL > 8 && (e = cudaFuncSetAttribute(k_ahp_mid_cl, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)) !=
                        cudaSuccess)
        return e;
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = CL;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.gridDim = dim3(4 * CL, 1, 1);
      cfg.blockDim = dim3(1024, 1, 1);
      cfg.dynamicSmemBytes = 0;
      cfg.stream = st;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      if ((e = cudaLaunchKernelEx(&cfg, k_ahp_mid_cl, g, d)) != cudaSuccess) return e;
    }
  }
  return cudaGetLastError();
}
cudaError_t launch_ahp_decide(bool fp64, const Geo& g, const Opt& o, int* state, const ReqsDev& R, const OutDev& O,
                              int r, const ShardDev& d, cudaStream_t st) {
  // FP32: PG over the grid, the last CTA decides (and commits); FP64: one CTA
  if (!fp64) k_ahp_pg<<<d.npart, 1024, 0, st>>>(g, o, state, R, O, r, d);
  else k_ahp_decide<true><<<1, 1024, 0, st>>>(g, o, state, R, O, r, d);
  return cudaGetLastError();
}
// After a request's last pod step (the host saw PH_DONE): the presorted orders re-merged on
// clusters (no-ops unless facc[14] was set by an accepted request's commit)
cudaError_t launch_presort_update(const Geo& g, const Opt& o, int* state, const ShardDev& d, cudaStream_t st) {
  cudaError_t e;
  const int CL = sh_levels_cluster();
  if (CL > 8 && (e = cudaFuncSetAttribute(k_presort_update_cl, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)) !=
                    cudaSuccess)
    return e;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(3 * CL, 1, 1);
  cfg.blockDim = dim3(1024, 1, 1);
  cfg.dynamicSmemBytes = sizeof(unsigned) * (size_t)((g.n + 31) / 32);
  cfg.stream = st;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if ((e = cudaLaunchKernelEx(&cfg, k_presort_update_cl, g, o, state, d)) != cudaSuccess) return e;
  k_presort_update_fin<<<1, 256, 0, st>>>(g, d);
  return cudaGetLastError();
}

size_t scratch_bytes() { return sizeof(Scratch); }



cudaError_t launch_sh_begin(const Geo& g, const Opt& o, int* state, const ReqsDev& R, const OutDev& O, int r,
                            const ShardDev& d, cudaStream_t st) {
  if (o.method == 1) {
    k_sh_begin<1><<<1, 1024, 0, st>>>(g, o, state, R, O, r, d, r == 0);
  } else {
    const int P2 = next_pow2(g.n), S = P2 < SQP_RUN ? P2 : SQP_RUN;
    const size_t sm = sizeof(unsigned long long) * (size_t)S;
    cudaError_t e = cudaFuncSetAttribute(k_presort_runs, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    k_presort_runs<<<3 * (P2 / S), 1024, sm, st>>>(g, state, d, r == 0);
    k_presort_merge<<<(3 * P2 + 255) / 256, 256, 0, st>>>(g, d, r == 0);
    k_sh_begin<0><<<1, 1024, 0, st>>>(g, o, state, R, O, r, d, 2);
  }
  return cudaGetLastError();
}
cudaError_t launch_sh_prep(const Geo& g, const Opt& o, int* state, const ReqsDev& R, const OutDev& O, int r,
                           const ShardDev& d, cudaStream_t st) {
  const int fgrid = (g.n + 1023) / 1024;
  if (o.method == 1) {
    k_sh_prep_a<1><<<1, 1024, 0, st>>>(g, o, state, R, O, r, d);
    k_sh_filter<1><<<fgrid, 1024, 0, st>>>(g, o, state, d);
  } else {
    k_sh_prep_a<0><<<1, 1024, 0, st>>>(g, o, state, R, O, r, d);
    k_sh_filter<0><<<fgrid, 1024, 0, st>>>(g, o, state, d);
  }
  const size_t bits = 2 * sizeof(unsigned) * (size_t)((g.n + 31) / 32);
  if (o.method == 1) {
    k_sh_prep<1><<<1, 1024, 0, st>>>(g, o, state, R, O, r, d);
  } else {
    const int CL = sh_levels_cluster();
    if (CL <= 1) {
      k_sh_prep<0><<<1, 1024, 0, st>>>(g, o, state, R, O, r, d);
      k_sh_levels<<<4, 1024, bits, st>>>(g, o, state, d);  // one CTA per criterion
    } else {  // a cluster of CL CTAs per criterion
      if (CL > 8) {
        cudaError_t e = cudaFuncSetAttribute(k_sh_levels_cl, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
      }
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = CL;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.gridDim = dim3(4 * CL, 1, 1);
      cfg.blockDim = dim3(1024, 1, 1);
      cfg.dynamicSmemBytes = bits;
      cfg.stream = st;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      // (k_sh_prep's work runs in the cluster kernel's CTA 0)
      cudaError_t e = cudaLaunchKernelEx(&cfg, k_sh_levels_cl, g, o, state, R, O, r, d);
      if (e != cudaSuccess) return e;
    }
  }
  return cudaGetLastError();
}
cudaError_t launch_sh_score(const Geo& g, const Opt& o, int* state, int lo, int hi, int slot, const ShardDev& d,
                            cudaStream_t st) {
  k_sh_score<<<1, 1024, 0, st>>>(g, o, state, lo, hi, slot, d);
  return cudaGetLastError();
}
cudaError_t launch_sh_decide(const Geo& g, const Opt& o, int* state, const ReqsDev& R, const OutDev& O, int r,
                             int world, const ShardDev& d, cudaStream_t st) {
  k_sh_decide<<<1, 1024, 0, st>>>(g, o, state, R, O, r, world, d);
  return cudaGetLastError();
}
cudaError_t launch_sh_fp64(const Geo& g, const Opt& o, int* state, int lo, int hi, int slot, const ShardDev& d,
                           cudaStream_t st) {
  k_sh_fp64<<<1, 1024, 0, st>>>(g, o, state, lo, hi, slot, d);
  return cudaGetLastError();
}
cudaError_t launch_sh_decide64(const Geo& g, const Opt& o, int* state, const ReqsDev& R, const OutDev& O, int r,
                               int world, const ShardDev& d, cudaStream_t st) {
  k_sh_decide64<<<1, 1024, 0, st>>>(g, o, state, R, O, r, world, d);
  return cudaGetLastError();
}

// ------------------------------------------------------------ departures ---
// nacs_release: the accepted requests' allocations return to
// the state — the exact inverse of commit + top-up.  Phase 1 accumulates per-word deltas
// (a thread per request, atomics) and checks each placement's structure; phase 2 checks
// residual <= capacity on every touched word; phase 3 applies the deltas and re-derives f_u
// of the touched servers (R22).  Nothing is applied when phase 1 or 2 found a violation.
__global__ void k_release_delta(Geo g, ReqsDev R, OutDev P, const int* idx, int n_idx, long long* delta,
                                int* bad) {
  const int n = g.n, h = g.h;
  const int cnt = idx ? n_idx : R.n;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < cnt; t += gridDim.x * blockDim.x) {
    const int r = idx ? idx[t] : t;
    if (P.status[r] != 1) continue;
    const int c0 = R.coff[r], c1 = R.coff[r + 1], v0 = R.voff[r], v1 = R.voff[r + 1];
    int b = 0;
    for (int i = c0; i < c1; ++i) {
      const int u = P.server[i];
      if (u < 0 || u >= n || P.cpu_a[i] < 0 || P.ram_a[i] < 0) { b = 1; continue; }
      atomicAdd(reinterpret_cast<unsigned long long*>(delta + u), (unsigned long long)(long long)P.cpu_a[i]);
      atomicAdd(reinterpret_cast<unsigned long long*>(delta + n + u), (unsigned long long)(long long)P.ram_a[i]);
    }
    for (int e = v0; e < v1; ++e) {
      const int a = R.src[e], d = R.dst[e], bw = P.bw_a[e], pid = P.path[e];
      if (a < 0 || a >= c1 - c0 || d < 0 || d >= c1 - c0 || bw < 0) { b = 1; continue; }
      const int us = P.server[c0 + a], ud = P.server[c0 + d];
      if (us < 0 || us >= n || ud < 0 || ud >= n) { b = 1; continue; }
      if (us == ud) {  // host bus: no link carried it
        if (pid != -1) b = 1;
        continue;
      }
      const int eu = us / h, ev = ud / h;
      const bool ok = eu == ev ? pid == 0 : (eu / h == ev / h ? (pid >= 1 && pid <= h) : (pid > h && pid <= h + h * h));
      if (!ok) { b = 1; continue; }
      int off[4];
      const int m = path_links(g, us, ud, pid, off);
      atomicAdd(reinterpret_cast<unsigned long long*>(delta + 3 * n + us), (unsigned long long)(long long)bw);
      atomicAdd(reinterpret_cast<unsigned long long*>(delta + 3 * n + ud), (unsigned long long)(long long)bw);
      for (int k = 0; k < m; ++k)
        atomicAdd(reinterpret_cast<unsigned long long*>(delta + off[k]), (unsigned long long)(long long)bw);
    }
    if (b) atomicOr(bad, 1);
  }
}

__device__ __forceinline__ long long word_cap(const Geo& g, int w) {
  return w < g.n ? g.cpu_cap : (w < 2 * g.n ? g.ram_cap : (w < 3 * g.n ? 1 : g.link_cap));
}

__global__ void k_release_check(Geo g, const int* state, const long long* delta, int* bad) {
  const int W = g.words();
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < W; w += gridDim.x * blockDim.x)
    if (delta[w] && (long long)state[w] + delta[w] > word_cap(g, w)) atomicOr(bad, 2);
}

__global__ void k_release_apply(Geo g, int* state, const long long* delta, const int* bad) {
  if (*bad) return;
  const int n = g.n, W = g.words();
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < W; w += gridDim.x * blockDim.x) {
    if (w < n) {
      if (delta[w] || delta[n + w]) {
        const int c = state[w] + (int)delta[w], r = state[n + w] + (int)delta[n + w];
        state[w] = c;
        state[n + w] = r;
        state[2 * n + w] = (c < g.cpu_cap || r < g.ram_cap) ? 1 : 0;
      }
    } else if (w >= 3 * n && delta[w]) {
      state[w] += (int)delta[w];
    }
  }
}

cudaError_t launch_release(const Geo& g, int* state, const ReqsDev& R, const OutDev& P, const int* idx, int n_idx,
                           long long* delta, int* bad, cudaStream_t st) {
  const int W = g.words();
  cudaError_t e = cudaMemsetAsync(delta, 0, sizeof(long long) * (size_t)W, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(bad, 0, sizeof(int), st);
  if (e != cudaSuccess) return e;
  const int cnt = idx ? n_idx : R.n;
  if (cnt > 0) k_release_delta<<<std::min(1184, (cnt + 127) / 128), 128, 0, st>>>(g, R, P, idx, n_idx, delta, bad);
  const int gw = std::min(1184, (W + 255) / 256);
  k_release_check<<<gw, 256, 0, st>>>(g, state, delta, bad);
  k_release_apply<<<gw, 256, 0, st>>>(g, state, delta, bad);
  return cudaGetLastError();
}

// Fragmentation counters of one simulator tick: active servers |N^s'| (f_u = 1)
// and active links |E^s'| (residual below capacity) into out[0], out[1] (zeroed by the caller).
__global__ void k_tick_counts(Geo g, const int* state, int* out) {
  int as = 0, al = 0;
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < g.n; u += gridDim.x * blockDim.x) as += state[2 * g.n + u];
  for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < g.L; l += gridDim.x * blockDim.x)
    al += state[3 * g.n + l] < g.link_cap ? 1 : 0;
  for (int o = 16; o; o >>= 1) {
    as += __shfl_xor_sync(0xFFFFFFFFu, as, o);
    al += __shfl_xor_sync(0xFFFFFFFFu, al, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (as) atomicAdd(out, as);
    if (al) atomicAdd(out + 1, al);
  }
}

cudaError_t launch_tick_counts(const Geo& g, const int* state, int* out, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(out, 0, 2 * sizeof(int), st);
  if (e != cudaSuccess) return e;
  k_tick_counts<<<std::min(148, (g.L + 255) / 256), 256, 0, st>>>(g, state, out);
  return cudaGetLastError();
}

// --------------------------------------------------------------- host -------
int batch_block_size(const Geo& g, int method) {
  if (method == 0) {  // AHP: a warp per level pair in the passes
    const char* e = getenv("NACS_AHP_BLOCK");
    if (e) return atoi(e);
    // about one (l, K-1-l) level pair per thread in the passes: warm snapshots leave
    // n_f ~ 0.6 n feasible, so ~0.3 n pairs; 7n/16 threads measured best at C3 (A/B over
    // 256..512 threads: 448 -> 44.8 ms, 512 -> 47.1 ms, 320 -> 45.1 ms, 256 -> 54.0 ms)
    int b = ((7 * g.n / 16 + 31) / 32) * 32;
    return b < 128 ? 128 : (b > 512 ? 512 : b);
  }
  int b = ((g.n / 8 + 31) / 32) * 32;  // about 8 servers per thread
  if (b < 64) b = 64;
  if (b > 1024) b = 1024;
  return b;
}

static size_t bitmap_bytes(const Geo& g) {
  int nW = (g.n + 31) / 32, nEW = (g.E + 31) / 32;
  return align16(4 * (size_t)nW) * 3 + align16(4 * (size_t)nEW);
}

// AHP whose sorted-level workspace (ahp_bytes, ~68 B per server) does not fit beside the
// snapshot (k = 32: 196 KB + 561 KB) keeps only the snapshot and bitmaps in shared memory and
// carves the workspace from a per-CTA block of global memory (L1/L2-resident).
bool batch_ahp_global(const Geo& g, int method) {
  if (method != 0) return false;
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const size_t b = align16(sizeof(int) * (size_t)g.words()) + bitmap_bytes(g) + sizeof(Scratch) + 64;
  return b + ahp_bytes(g.n) > (size_t)optin && b <= (size_t)optin;
}

size_t batch_smem_bytes(const Geo& g, int method) {
  size_t b = align16(sizeof(int) * (size_t)g.words()) + bitmap_bytes(g);
  if (method == 0 && !batch_ahp_global(g, method)) b += ahp_bytes(g.n);
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (b + sizeof(Scratch) + 64 > (size_t)optin) return 0;
  return b;
}

template <int M>
static cudaError_t batch_occupancy_t(const Geo& g, int* blocks_per_sm) {
  size_t smem = batch_smem_bytes(g, M);
  if (!smem) { *blocks_per_sm = 0; return cudaSuccess; }
  cudaError_t e = cudaFuncSetAttribute(k_batch<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, k_batch<M>, batch_block_size(g, M), smem);
}

cudaError_t batch_occupancy(const Geo& g, int method, int* blocks_per_sm) {
  switch (method) {
    case 0: return batch_occupancy_t<0>(g, blocks_per_sm);
    case 1: return batch_occupancy_t<1>(g, blocks_per_sm);
    case 2: return batch_occupancy_t<2>(g, blocks_per_sm);
    default: return batch_occupancy_t<3>(g, blocks_per_sm);
  }
}

template <int M>
static void launch_batch_t(const Geo& g, const Opt& o, const int* d_state, const ReqsDev& R, const OutDev& O,
                           int2* ulog, double* w64, unsigned char* ahp_g, int* next, unsigned long long* stats,
                           int grid, cudaStream_t st, const int* idx, const int* n_idx) {
  size_t smem = batch_smem_bytes(g, M);
  if (M == 0 && ahp_g) {
    cudaFuncSetAttribute(k_batch<M, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_batch<M, true><<<grid, batch_block_size(g, M), smem, st>>>(g, o, d_state, R, O, ulog, w64, ahp_g, next, stats,
                                                                 idx, n_idx);
    return;
  }
  cudaFuncSetAttribute(k_batch<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_batch<M><<<grid, batch_block_size(g, M), smem, st>>>(g, o, d_state, R, O, ulog, w64, ahp_g, next, stats, idx,
                                                         n_idx);
}

cudaError_t launch_batch(const Geo& g, const Opt& o, const int* d_state, const ReqsDev& R, const OutDev& O,
                         int2* ulog, double* w64, unsigned char* ahp_g, int* next, unsigned long long* stats,
                         int grid, cudaStream_t st, const int* idx, const int* n_idx) {
  switch (o.method) {
    case 0: launch_batch_t<0>(g, o, d_state, R, O, ulog, w64, ahp_g, next, stats, grid, st, idx, n_idx); break;
    case 1: launch_batch_t<1>(g, o, d_state, R, O, ulog, w64, nullptr, next, stats, grid, st, idx, n_idx); break;
    case 2: launch_batch_t<2>(g, o, d_state, R, O, ulog, w64, nullptr, next, stats, grid, st, idx, n_idx); break;
    default: launch_batch_t<3>(g, o, d_state, R, O, ulog, w64, nullptr, next, stats, grid, st, idx, n_idx); break;
  }
  return cudaGetLastError();
}

static int single_block_size(const Geo& g) {
  if (const char* e = getenv("NACS_SEQ_BLOCK")) return atoi(e);  // experiments
  int b = ((g.n / 4 + 31) / 32) * 32;
  if (b < 64) b = 64;
  if (b > 1024) b = 1024;
  return b;
}

// dynamic shared memory of the sequential kernels: bitmaps, plus the live state when it fits
static size_t seq_smem_bytes(const Geo& g, int* smem_state) {
  const size_t b = bitmap_bytes(g), st = align16(sizeof(int) * (size_t)g.words());
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  *smem_state = b + st + sizeof(Scratch) + 1024 <= (size_t)optin;
  return *smem_state ? b + st : b;
}

template <int M, class K>
static void set_smem(K kernel, size_t smem) {
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

cudaError_t launch_sequential(const Geo& g, const Opt& o, int* d_state, const ReqsDev& R, const OutDev& O,
                              int2* ulog, float* ahp_ws, double* w64, unsigned long long* stats,
                              cudaStream_t st) {
  int ss = 0;
  const size_t smem = seq_smem_bytes(g, &ss);
  int B = single_block_size(g);
  switch (o.method) {
    case 0: set_smem<0>(k_sequential<0>, smem); k_sequential<0><<<1, B, smem, st>>>(g, o, d_state, R, O, ulog, ahp_ws, w64, stats, ss); break;
    case 1: set_smem<1>(k_sequential<1>, smem); k_sequential<1><<<1, B, smem, st>>>(g, o, d_state, R, O, ulog, ahp_ws, w64, stats, ss); break;
    case 2: set_smem<2>(k_sequential<2>, smem); k_sequential<2><<<1, B, smem, st>>>(g, o, d_state, R, O, ulog, ahp_ws, w64, stats, ss); break;
    default: set_smem<3>(k_sequential<3>, smem); k_sequential<3><<<1, B, smem, st>>>(g, o, d_state, R, O, ulog, ahp_ws, w64, stats, ss); break;
  }
  return cudaGetLastError();
}

int seq_cluster_size(const Geo& g) {
  if (const char* e = getenv("NACS_SEQC")) {  // experiments (0 = off)
    const int C = atoi(e);  // a power of two (mirror_ptr)
    return C > 0 && C <= 16 && !(C & (C - 1)) && (long long)C * SQC_M >= g.n ? C : 0;
  }
  if (g.n < 16384 || g.n > 65536) return 0;  // below: the one-CTA engine keeps the state in shared memory
  return g.n > 32768 ? 16 : 8;  // at most SQC_M servers per CTA
}

cudaError_t launch_seq_cluster(const Geo& g, const Opt& o, int* d_state, const ReqsDev& R, const OutDev& O,
                               int2* ulog, unsigned long long* stats, unsigned long long* work, int C,
                               cudaStream_t st) {
  // work: facc [2][16] | kx [2][16] | kxv [16] | kxi [16] (unsigned long long words)
  unsigned long long* facc = work;
  unsigned long long* kx = work + 32;
  double* kxv = reinterpret_cast<double*>(work + 64);
  int* kxi = reinterpret_cast<int*>(work + 80);
  const size_t nW = (size_t)(g.n + 31) / 32, nEW = (size_t)(g.E + 31) / 32;
  const size_t smem = 4 * align16(4 * nW) + align16(4 * nEW) + sizeof(int) * 4 * SQC_M;
  cudaError_t e;
  if (C > 8 && (e = cudaFuncSetAttribute(k_seq_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)) !=
                   cudaSuccess)
    return e;
  if ((e = cudaFuncSetAttribute(k_seq_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess)
    return e;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(C, 1, 1);
  cfg.blockDim = dim3(SQC_T, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_seq_cluster, g, o, d_state, R, O, ulog, stats, facc, kx, kxv, kxi);
}

cudaError_t launch_simulate(const Geo& g, const Opt& o, int* d_state, const ReqsDev& R, const OutDev& O,
                            int2* ulog, float* ahp_ws, double* w64, unsigned long long* stats, const SimDev& S,
                            cudaStream_t st) {
  int ss = 0;
  const size_t smem = seq_smem_bytes(g, &ss);
  const int B = std::min(512, single_block_size(g));  // k_simulate: __launch_bounds__(512)
  switch (o.method) {
    case 0: set_smem<0>(k_simulate<0>, smem); k_simulate<0><<<1, B, smem, st>>>(g, o, d_state, R, O, ulog, ahp_ws, w64, stats, S, ss); break;
    case 1: set_smem<1>(k_simulate<1>, smem); k_simulate<1><<<1, B, smem, st>>>(g, o, d_state, R, O, ulog, ahp_ws, w64, stats, S, ss); break;
    case 2: set_smem<2>(k_simulate<2>, smem); k_simulate<2><<<1, B, smem, st>>>(g, o, d_state, R, O, ulog, ahp_ws, w64, stats, S, ss); break;
    default: set_smem<3>(k_simulate<3>, smem); k_simulate<3><<<1, B, smem, st>>>(g, o, d_state, R, O, ulog, ahp_ws, w64, stats, S, ss); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_rank(const Geo& g, const Opt& o, int* d_state, const QueryDev& q, float* ahp_ws, double* w64,
                        unsigned long long* stats, cudaStream_t st) {
  size_t smem = bitmap_bytes(g);
  int B = single_block_size(g);
  if (o.method == 1) k_rank<1><<<1, B, smem, st>>>(g, o, d_state, q, ahp_ws, w64, stats);
  else k_rank<0><<<1, B, smem, st>>>(g, o, d_state, q, ahp_ws, w64, stats);
  return cudaGetLastError();
}

// ------------------------------------------------ logical bandwidth criterion ---
// R2's alternative reading (`bw_criterion = logical`, "the sum of all bandwidth
// capacity bw^s_uv with source on u"): L(u) = sum over servers v != u of the bottleneck of
// the widest shortest u-v path on the current state, min(acc_u, acc_v, F(e_u, e_v)) with
// F the widest fabric bottleneck between the two edge switches (R16; +inf on one switch).
// k_ft_fabric: F for every ordered pair of edge switches (a thread per pair, h or h^2 paths);
// k_ft_logical: a CTA per edge switch sums min(.) over all servers for its h servers.
__global__ void k_ft_fabric(Geo g, const int* __restrict__ state, int* F) {
  const int E = g.E, h = g.h, n = g.n;
  const int* EA = state + 4 * n;
  const int* AC = EA + E * h;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < E * E; idx += gridDim.x * blockDim.x) {
    const int e = idx / E, f = idx - e * E;
    int best;
    if (e == f) {
      best = INT_MAX;
    } else if (e / h == f / h) {
      best = 0;
      for (int a = 0; a < h; ++a) best = max(best, min(EA[e * h + a], EA[f * h + a]));
    } else {
      const int pe = e / h, pf = f / h;
      best = 0;
      for (int a = 0; a < h; ++a) {
        const int up = min(EA[e * h + a], EA[f * h + a]);
        if (up <= best) continue;
        for (int b = 0; b < h; ++b)
          best = max(best, min(up, min(AC[(pe * h + a) * h + b], AC[(pf * h + a) * h + b])));
      }
    }
    F[idx] = best;
  }
}

__global__ void __launch_bounds__(256) k_ft_logical(Geo g, const int* __restrict__ state, const int* __restrict__ F,
                                                    int* crit, int* too_big) {
  const int e = blockIdx.x, h = g.h, n = g.n;
  const int* acc = state + 3 * n;
  __shared__ long long part[8][32];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = 0; i < h; ++i) {
    const int u = e * h + i;
    const int au = acc[u];
    long long sum = 0;
    for (int v = threadIdx.x; v < n; v += blockDim.x) {
      if (v == u) continue;
      sum += min(min(au, acc[v]), F[e * g.E + v / h]);
    }
    for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xFFFFFFFFu, sum, o);
    if (lane == 0) part[w][i] = sum;
  }
  __syncthreads();
  if (threadIdx.x < h) {
    long long L = 0;
    for (int j = 0; j < (int)(blockDim.x >> 5); ++j) L += part[j][threadIdx.x];
    if (L >= (1LL << 24)) atomicOr(too_big, 1);  // not exact in FP32 (R5): the caller fails
    crit[3 * n + e * h + threadIdx.x] = (int)min(L, (long long)INT_MAX);
  }
}

cudaError_t launch_logical_criteria(const Geo& g, const int* state, int* crit, int* F, int* too_big,
                                    cudaStream_t st) {
  cudaError_t e = cudaMemcpyAsync(crit, state, sizeof(int) * 3 * (size_t)g.n, cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(too_big, 0, sizeof(int), st);
  if (e != cudaSuccess) return e;
  const int EE = g.E * g.E;
  k_ft_fabric<<<std::min(4096, (EE + 255) / 256), 256, 0, st>>>(g, state, F);
  k_ft_logical<<<g.E, 256, 0, st>>>(g, state, F, crit, too_big);
  return cudaGetLastError();
}

size_t ahp_workspace_bytes(int n) { return ahp_bytes(n); }
size_t ahp_workspace_doubles(int n) { return ahp_w64_doubles(n); }

cudaError_t launch_validate(const ReqsDev& R, int* status, unsigned long long* stats, cudaStream_t st) {
  if (R.n <= 0) return cudaSuccess;
  k_validate<<<(R.n + 255) / 256, 256, 0, st>>>(R, status, stats);
  return cudaGetLastError();
}

}  // namespace nacs
