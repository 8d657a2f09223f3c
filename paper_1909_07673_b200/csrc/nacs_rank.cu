// nacs_rank.cu — whole-GPU TOPSIS ranking of one pod step on one or many DC states
// (§8(d) "standalone nacs_rank_topsis on cold snapshots").
//
// One THREAD-BLOCK CLUSTER ranks one DC state: the C = ceil(n / 4096) CTAs of the cluster
// each own a slice of <= 4096 servers (512 threads x 8 servers, loaded once with coalesced
// streaming vector loads and kept in registers for every pass).  Per state:
//   a2  fabric feasibility of the slice's edge switches for every flow (shared memory),
//   a3+a4 filter + exact integer statistics of the slice   -> DSMEM exchange (cluster.sync)
//   a5T FP32 closeness, scores/mask written, top-2 keys    -> DSMEM exchange
//   a7  argmax; near ties re-decided in FP64 on the registers -> DSMEM exchange.
// Every CTA of a cluster reduces the C partials in the same rank order, so all of them take
// the same decision without a second round trip.  A persistent grid of clusters walks the
// states (state b -> cluster b mod #clusters), so a single call streams B states at HBM rate:
// the algorithmic traffic is 16 B read per server (cpu, ram, f_u, access link) plus the
// 4 B score (and 1 B mask) written.  Paper: TOPSIS P:365-375 (R12-R13), filter Eq. 4-7
// P:181-189 (R6), "parallel reduction" P:380.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cfloat>
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

struct RmStats {  // one CTA's partial statistics over its slice (read by the cluster over DSMEM)
  unsigned long long q[3];
  int nf, nact, mn[3], mx[3], bad;
};
struct RmKeys {
  unsigned long long k1, k2;
};
struct RmArg {
  double v;
  int j;
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
__device__ __forceinline__ void stm(uint8_t* p, const bool (&x)[4]) {
  *reinterpret_cast<unsigned*>(p) = (x[0] ? 1u : 0u) | (x[1] ? 1u << 8 : 0u) | (x[2] ? 1u << 16 : 0u) |
                                    (x[3] ? 1u << 24 : 0u);
}
__device__ __forceinline__ void stm(uint8_t* p, const bool (&x)[2]) {
  *reinterpret_cast<unsigned short*>(p) = (unsigned short)((x[0] ? 1u : 0u) | (x[1] ? 1u << 8 : 0u));
}

}  // namespace

// Per-CTA shared state of k_rank_many.
struct RmShared {
  RmStats st;
  RmKeys keys;
  RmArg arg;
  unsigned edgebad[RM_EW];      // slice edge e (relative to the slice's first edge): some flow fails
  unsigned special[RM_S / 32];  // slice server: a flow server or an excluded server
  unsigned pm[MAXK];            // a2 scratch: per fat-tree pod, bit a = core route via agg a ok
  unsigned vm;                  // a2 scratch: the flow server's edge uplinks >= D
  int fv[MAXF], fD[MAXF];
  int fok[MAXF], fexcl[MAXF];
  int sumD, G;
  int red_i[RM_NW][8];
  unsigned long long red_u[RM_NW][3];
  unsigned long long red_k[RM_NW][2];
  double red_d[RM_NW];
  int red_j[RM_NW];
};

// grid = #clusters x C CTAs, cluster dims (C, 1, 1) set at launch
template <int VW>
__global__ void __launch_bounds__(RM_T, 1) k_rank_many(RankManyArgs a) {
  __shared__ RmShared sm;
  cg::cluster_group cl = cg::this_cluster();
  const int C = (int)cl.num_blocks();
  const int rank = (int)cl.block_rank();
  const int ncl = gridDim.x / C;
  const int cid = blockIdx.x / C;
  const Geo& g = a.g;
  const int n = g.n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int S = a.slice;
  const int lo = rank * S, hi = min(n, lo + S);
  const bool net = a.path_filter && a.nflow > 0;
  const int e_lo = lo < hi ? (int)div_h((unsigned)lo, g.magic_h) : 0;
  const int e_hi = lo < hi ? (int)div_h((unsigned)(hi - 1), g.magic_h) : -1;
  constexpr int NJ = RM_V / VW;

  // a0: the slice's criteria rows, in registers; the next state's rows are loaded while this
  // state is ranked (software pipelining: the loads stay in flight across the cluster syncs)
  int x[NJ][4][VW], xn[NJ][4][VW];
  auto load = [&](int bb, int (&y)[NJ][4][VW]) {
    const int* sp = a.states + (long long)bb * a.stride;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int u0 = lo + VW * (tid + RM_T * j);
      if (u0 < hi) {
#pragma unroll
        for (int c = 0; c < 4; ++c) ldv(sp + c * n + u0, y[j][c]);
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int v = 0; v < VW; ++v) y[j][c][v] = 0;
      }
    }
  };
  if (cid < a.B) load(cid, x);
  for (int b = cid; b < a.B; b += ncl) {
    const int* st = a.states + (long long)b * a.stride;
    const int* EA = st + 4 * n;
    const int* AC = EA + g.E * g.h;
    if (b + ncl < a.B) load(b + ncl, xn);
    // ------------------------------------------ flows: a2 fabric, special servers --
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
    if (net && lo < hi) {
      const int h = g.h;
      const int p_lo = (int)div_h((unsigned)e_lo, g.magic_h), p_hi = (int)div_h((unsigned)e_hi, g.magic_h);
      for (int f = 0; f < a.nflow; ++f) {
        const int v = sm.fv[f], D = sm.fD[f];
        const int ev = (int)div_h((unsigned)v, g.magic_h), pv = (int)div_h((unsigned)ev, g.magic_h);
        // pm[p] bit a: some core (a, b) joins pod p and pod pv with both links >= D
        for (int p = p_lo + tid; p <= p_hi; p += RM_T) sm.pm[p] = 0u;
        if (tid == 0) sm.vm = 0u;
        __syncthreads();
        for (int t = tid; t < (p_hi - p_lo + 1) * h; t += RM_T) {
          const int pr = (int)div_h((unsigned)t, g.magic_h), aa = t - pr * h, p = p_lo + pr;
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
        for (int e = e_lo + tid; e <= e_hi; e += RM_T) {
          if (e == ev) continue;  // same edge switch: access links only
          unsigned em = 0;
          for (int aa = 0; aa < h; ++aa) em |= (EA[e * h + aa] >= D ? 1u : 0u) << aa;
          const int pe = (int)div_h((unsigned)e, g.magic_h);
          const unsigned ok = pe == pv ? (em & vm) : (em & vm & sm.pm[pe]);
          if (!ok) atomicOr(&sm.edgebad[(e - e_lo) >> 5], 1u << ((e - e_lo) & 31));
        }
        __syncthreads();
      }
    }
    // flow servers and excluded servers of the slice (R17 host-bus flows, R18 exclusions)
    if (tid < a.nflow) {
      const int f = tid, u = sm.fv[f];
      if (u >= lo && u < hi) {
        bool ok = st[3 * n + u] >= sm.sumD - sm.fD[f];
        for (int o = 0; o < a.nflow; ++o)
          if (o != f && st[3 * n + sm.fv[o]] < sm.fD[o]) ok = false;
        const int e = (int)div_h((unsigned)u, g.magic_h);
        if (net && ((sm.edgebad[(e - e_lo) >> 5] >> ((e - e_lo) & 31)) & 1u)) ok = false;
        sm.fok[f] = ok;
        atomicOr(&sm.special[(u - lo) >> 5], 1u << ((u - lo) & 31));
      }
    }
    __syncthreads();
    for (int i = tid; i < a.nex; i += RM_T) {
      const int u = a.ex[i];
      if (u >= lo && u < hi) atomicOr(&sm.special[(u - lo) >> 5], 1u << ((u - lo) & 31));
      for (int f = 0; f < a.nflow; ++f)
        if (sm.fv[f] == u) sm.fexcl[f] = 1;
    }
    __syncthreads();
    // --------------------------------------------------- a3 + a4: filter, stats --
    bool ok[NJ][VW];
    int nf = 0, nact = 0, bad = 0;
    unsigned mn0 = UINT_MAX, mn1 = UINT_MAX, mn3 = UINT_MAX, mx0 = 0, mx1 = 0, mx3 = 0;
    unsigned long long q0 = 0, q1 = 0, q3 = 0;
    const bool G = sm.G != 0;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int u0 = lo + VW * (tid + RM_T * j);
#pragma unroll
      for (int v = 0; v < VW; ++v) {
        const int u = u0 + v;
        const bool in = u < hi;
        const int x0 = x[j][0][v], x1 = x[j][1][v], x2 = x[j][2][v], x3 = x[j][3][v];
        // R5: every value must be an exact FP32 integer in range (device-pointer states are
        // validated here; a violation invalidates the state's result)
        if (in && ((unsigned)x0 > (unsigned)g.cpu_cap || (unsigned)x1 > (unsigned)g.ram_cap ||
                   (unsigned)x2 > 1u || (unsigned)x3 > (unsigned)g.link_cap))
          bad = 1;
        bool k = in && x0 >= a.dc && x1 >= a.dr;
        if (net) {
          const int e = (int)div_h((unsigned)u, g.magic_h) - e_lo;
          k = k && G && x3 >= sm.sumD && !((sm.edgebad[e >> 5] >> (e & 31)) & 1u);
        }
        if (in && ((sm.special[(u - lo) >> 5] >> ((u - lo) & 31)) & 1u)) {
          int f = -1;
          for (int i = 0; i < a.nflow; ++i) if (sm.fv[i] == u) f = i;
          k = f >= 0 && !sm.fexcl[f] && x0 >= a.dc && x1 >= a.dr && (!a.path_filter || sm.fok[f]);
        }
        ok[j][v] = k;
        if (k) {
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
    }
    nf = (int)__reduce_add_sync(NACS_FULL, (unsigned)nf);
    nact = (int)__reduce_add_sync(NACS_FULL, (unsigned)nact);
    bad = (int)__reduce_or_sync(NACS_FULL, (unsigned)bad);
    mn0 = __reduce_min_sync(NACS_FULL, mn0); mx0 = __reduce_max_sync(NACS_FULL, mx0);
    mn1 = __reduce_min_sync(NACS_FULL, mn1); mx1 = __reduce_max_sync(NACS_FULL, mx1);
    mn3 = __reduce_min_sync(NACS_FULL, mn3); mx3 = __reduce_max_sync(NACS_FULL, mx3);
    q0 = warp_sum_u64(q0);
    q1 = warp_sum_u64(q1);
    q3 = warp_sum_u64(q3);
    if (lane == 0) {
      int* r = sm.red_i[warp];
      r[0] = nf; r[1] = nact; r[2] = (int)mn0; r[3] = (int)mx0; r[4] = (int)mn1; r[5] = (int)mx1;
      r[6] = (int)mn3; r[7] = (int)mx3 | (bad << 31);
      sm.red_u[warp][0] = q0; sm.red_u[warp][1] = q1; sm.red_u[warp][2] = q3;
    }
    __syncthreads();
    if (warp == 0) {
      const bool in = lane < RM_NW;
      const int* r = sm.red_i[in ? lane : 0];
      nf = in ? r[0] : 0; nact = in ? r[1] : 0;
      mn0 = in ? (unsigned)r[2] : UINT_MAX; mx0 = in ? (unsigned)r[3] : 0;
      mn1 = in ? (unsigned)r[4] : UINT_MAX; mx1 = in ? (unsigned)r[5] : 0;
      mn3 = in ? (unsigned)r[6] : UINT_MAX; mx3 = in ? (unsigned)r[7] & 0x7fffffffu : 0;
      bad = in ? (int)((unsigned)r[7] >> 31) : 0;
      q0 = in ? sm.red_u[lane][0] : 0; q1 = in ? sm.red_u[lane][1] : 0; q3 = in ? sm.red_u[lane][2] : 0;
      nf = (int)__reduce_add_sync(NACS_FULL, (unsigned)nf);
      nact = (int)__reduce_add_sync(NACS_FULL, (unsigned)nact);
      bad = (int)__reduce_or_sync(NACS_FULL, (unsigned)bad);
      mn0 = __reduce_min_sync(NACS_FULL, mn0); mx0 = __reduce_max_sync(NACS_FULL, mx0);
      mn1 = __reduce_min_sync(NACS_FULL, mn1); mx1 = __reduce_max_sync(NACS_FULL, mx1);
      mn3 = __reduce_min_sync(NACS_FULL, mn3); mx3 = __reduce_max_sync(NACS_FULL, mx3);
      q0 = warp_sum_u64(q0);
      q1 = warp_sum_u64(q1);
      q3 = warp_sum_u64(q3);
      if (lane == 0) {
        sm.st.nf = nf; sm.st.nact = nact; sm.st.bad = bad;
        sm.st.mn[0] = (int)mn0; sm.st.mx[0] = (int)mx0;
        sm.st.mn[1] = (int)mn1; sm.st.mx[1] = (int)mx1;
        sm.st.mn[2] = (int)mn3; sm.st.mx[2] = (int)mx3;
        sm.st.q[0] = q0; sm.st.q[1] = q1; sm.st.q[2] = q3;
      }
    }
    cl.sync();  // (1) every slice's statistics are visible over DSMEM
    // the cluster totals, reduced in rank order by every CTA (exact integers)
    TopsisP tp;
    unsigned long long sq[4];
    int NF = 0, NACT = 0, BAD = 0;
    {
      unsigned m0 = UINT_MAX, m1 = UINT_MAX, m3 = UINT_MAX, M0 = 0, M1 = 0, M3 = 0;
      unsigned long long s0 = 0, s1 = 0, s3 = 0;
      for (int r = 0; r < C; ++r) {
        const RmStats* p = cl.map_shared_rank(&sm.st, r);
        NF += p->nf; NACT += p->nact; BAD |= p->bad;
        m0 = min(m0, (unsigned)p->mn[0]); M0 = max(M0, (unsigned)p->mx[0]);
        m1 = min(m1, (unsigned)p->mn[1]); M1 = max(M1, (unsigned)p->mx[1]);
        m3 = min(m3, (unsigned)p->mn[2]); M3 = max(M3, (unsigned)p->mx[2]);
        s0 += p->q[0]; s1 += p->q[1]; s3 += p->q[2];
      }
      tp.mn[0] = (int)m0; tp.mx[0] = (int)M0;
      tp.mn[1] = (int)m1; tp.mx[1] = (int)M1;
      tp.mn[2] = NACT == NF ? 1 : 0; tp.mx[2] = NACT > 0 ? 1 : 0;  // f_u in {0,1}
      tp.mn[3] = (int)m3; tp.mx[3] = (int)M3;
      sq[0] = s0; sq[1] = s1; sq[2] = (unsigned long long)NACT; sq[3] = s3;
    }
    topsis_params(tp, a.wd, sq);
    // ----------------------------------------------- a5T: closeness, top-2 keys --
    unsigned long long k1 = 0, k2 = 0;
    const bool live = NF > 0 && !BAD;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int u0 = lo + VW * (tid + RM_T * j);
      float sc[VW];
#pragma unroll
      for (int v = 0; v < VW; ++v) {
        sc[v] = 0.f;
        if (live && ok[j][v]) {
          sc[v] = topsis32(tp, x[j][0][v], x[j][1][v], x[j][2][v], x[j][3][v]);
          top2_insert(k1, k2, score_key(sc[v], u0 + v));
        }
      }
      if (u0 < hi) {
        if (a.scores) stv(a.scores + (long long)b * n + u0, sc);
        if (a.mask) {
          bool m[VW];
#pragma unroll
          for (int v = 0; v < VW; ++v) m[v] = ok[j][v] && !BAD;
          stm(a.mask + (long long)b * n + u0, m);
        }
      }
    }
    warp_top2(k1, k2);
    if (lane == 0) { sm.red_k[warp][0] = k1; sm.red_k[warp][1] = k2; }
    __syncthreads();
    if (warp == 0) {
      k1 = lane < RM_NW ? sm.red_k[lane][0] : 0ull;
      k2 = lane < RM_NW ? sm.red_k[lane][1] : 0ull;
      warp_top2(k1, k2);
      if (lane == 0) { sm.keys.k1 = k1; sm.keys.k2 = k2; }
    }
    cl.sync();  // (2) every slice's top-2 keys are visible
    unsigned long long K1 = 0, K2 = 0;
    for (int r = 0; r < C; ++r) {
      const RmKeys* p = cl.map_shared_rank(&sm.keys, r);
      top2_merge(K1, K2, p->k1, p->k2);
    }
    int best = K1 ? (int)(0xFFFFFFFFu - (unsigned)(K1 & 0xFFFFFFFFull)) : -1;
    const float s1 = __uint_as_float((unsigned)(K1 >> 32));
    const float s2 = __uint_as_float((unsigned)(K2 >> 32));
    const bool amb = live && K1 && (a.exact64 || (K2 != 0ull && s1 - s2 <= kTopsisDelta));
    if (amb) {  // FP64 re-decision over the near-max candidates (R14), on the registers
      const float thr = a.exact64 ? -1.0f : s1 - 2.0f * kTopsisDelta;
      double bv = -DBL_MAX;
      int bj = -1;
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const int u0 = lo + VW * (tid + RM_T * j);
#pragma unroll
        for (int v = 0; v < VW; ++v) {
          if (!ok[j][v]) continue;
          const int x0 = x[j][0][v], x1 = x[j][1][v], x2 = x[j][2][v], x3 = x[j][3][v];
          if (topsis32(tp, x0, x1, x2, x3) < thr) continue;
          const double r = topsis64(tp, x0, x1, x2, x3);
          if (r > bv || (r == bv && u0 + v < bj)) { bv = r; bj = u0 + v; }
        }
      }
      warp_argmax64(bv, bj);
      if (lane == 0) { sm.red_d[warp] = bv; sm.red_j[warp] = bj; }
      __syncthreads();
      if (warp == 0) {
        bv = lane < RM_NW ? sm.red_d[lane] : -DBL_MAX;
        bj = lane < RM_NW ? sm.red_j[lane] : -1;
        warp_argmax64(bv, bj);
        if (lane == 0) { sm.arg.v = bv; sm.arg.j = bj; }
      }
      cl.sync();  // (3) every slice's FP64 candidate is visible
      double BV = -DBL_MAX;
      int BJ = -1;
      for (int r = 0; r < C; ++r) {
        const RmArg* p = cl.map_shared_rank(&sm.arg, r);
        if (p->j >= 0 && (p->v > BV || (p->v == BV && p->j < BJ))) { BV = p->v; BJ = p->j; }
      }
      best = BJ;
    }
    if (rank == 0 && tid == 0) {
      a.best[b] = BAD ? -2 : (NF > 0 ? best : -1);
      if (a.stats) {
        atomicAdd(&a.stats[ST_POD_STEPS], 1ull);
        atomicAdd(&a.stats[ST_FEAS], (unsigned long long)NF);
        if (amb) atomicAdd(&a.stats[ST_FP64], 1ull);
        if (BAD) atomicAdd(&a.stats[ST_INVALID], 1ull);
      }
    }
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int v = 0; v < VW; ++v) x[j][c][v] = xn[j][c][v];
  }
  // no CTA may leave while another still reads its shared memory
  cl.sync();
}

// ------------------------------------------------------------------ host ---
int rank_many_cluster(const Geo& g) { return (g.n + RM_S - 1) / RM_S; }

cudaError_t launch_rank_many(const RankManyArgs& a0, int num_sms, cudaStream_t st) {
  RankManyArgs a = a0;
  const int C = rank_many_cluster(a.g);
  if (C > 16) return cudaErrorInvalidValue;
  const bool v4 = (a.g.n % 4 == 0) && (a.stride % 4 == 0);
  const int VW = v4 ? 4 : 2;
  // slices of <= RM_S servers, a multiple of VW so that vector accesses stay aligned
  int S = (a.g.n + C - 1) / C;
  S = (S + VW - 1) / VW * VW;
  a.slice = S;
  void (*kern)(RankManyArgs) = v4 ? k_rank_many<4> : k_rank_many<2>;
  static int max_clusters[2][17] = {};
  int& mc = max_clusters[v4][C];
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(RM_T, 1, 1);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e;
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
