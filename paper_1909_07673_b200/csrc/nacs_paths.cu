// nacs_paths.cu — general-topology widest-shortest paths: the "modified Dijkstra" of
// PAPER.md §V-D for DCs that are not fat-trees, and the
// logical-bandwidth criterion it enables (reading R2's alternative).
//
// Semantics (reading R26): a link is usable by a flow of demand D iff its
// residual >= D; the path has the fewest hops over usable links, then the largest
// bottleneck, then the lexicographically smallest vertex sequence.
//
// B200 design: one warp per query, level-synchronous BFS from the
// destination, every vertex labelled with ONE 32-bit key = (level mod 256) << 24 |
// (2^24 - 1 - width), so "fewer hops, then wider" is a single unsigned atomicMin in shared
// memory.  Levels are exact mod 256 because adjacent vertices differ by at most one level.
// Frontier vertices of small degree are expanded by their own lane; vertices of larger
// degree by the whole warp (one edge per lane), so a fat-tree switch level keeps 20 of 32
// lanes busy instead of serialising 20 dependent loads in one lane.  The walk from the
// source takes, per hop, the smallest-id neighbour one level closer whose label keeps the
// optimal bottleneck (a warp min-reduction).
//
// Two layouts, chosen at nacs_load_graph time:
//   SMEM: the whole CSR graph lives in shared memory, packed 4 bytes per adjacency entry
//         (neighbour:16 | residual:16; needs V <= 65536 and residuals <= 65535), with
//         per-warp key[V] (u32) and queue[V] (u16) beside it — every BFS access is on-chip.
//         The paper's DC (fat-tree k=20: 2500 vertices, 12000 entries) takes 58 KB.
//   GLOBAL: graph (int2 entries) read through L1/L2, per-warp scratch in shared memory when
//         it fits, else in global memory.
#include <algorithm>
#include <climits>
#include <cstdint>

#include "nacs_internal.h"

namespace nacs {

namespace {

constexpr unsigned UNVIS = 0xFFFFFFFFu;  // key of an unvisited vertex
constexpr unsigned WINF = 0xFFFFFFu;     // width of the root ("infinite"); residuals < 2^23
constexpr unsigned FULL = 0xFFFFFFFFu;
constexpr int HEAVY = 6;                 // degree above which the warp expands a vertex together

__device__ __forceinline__ unsigned width_of(unsigned key) { return WINF - (key & WINF); }

// Graph accessors: edge j = (neighbour, residual).
struct GlobalGraph {
  const int* off;
  const int2* adj;
  __device__ __forceinline__ int begin(int v) const { return __ldg(off + v); }
  __device__ __forceinline__ int end(int v) const { return __ldg(off + v + 1); }
  __device__ __forceinline__ int2 edge(int j) const { return __ldg(adj + j); }
};
struct SmemGraph {
  const int* off;        // shared
  const unsigned* adj;   // shared, neighbour | residual << 16
  __device__ __forceinline__ int begin(int v) const { return off[v]; }
  __device__ __forceinline__ int end(int v) const { return off[v + 1]; }
  __device__ __forceinline__ int2 edge(int j) const {
    const unsigned a = adj[j];
    return make_int2((int)(a & 0xFFFFu), (int)(a >> 16));
  }
};

// Per-warp scratch: key[V], queue[V] (u16 in SMEM mode), tail counter.
template <class QT>
struct Scratch2 {
  unsigned* key;
  QT* queue;
  int* tail;
};

// Relax edge (v -> a.x) of a level-`level` vertex with width Wv: label a.x at level nl.
// Returns true if a.x was unvisited before (the caller appends it to the queue).
__device__ __forceinline__ bool relax(unsigned* key, int2 a, unsigned Wv, unsigned nl, int demand) {
  if (a.y < demand) return false;  // link not usable for this demand (R26)
  const unsigned kw = ((volatile unsigned*)key)[a.x];
  if (kw != UNVIS && (kw >> 24) != nl) return false;  // settled at this or an earlier level
  const unsigned w = min((unsigned)a.y, Wv);
  return atomicMin(&key[a.x], (nl << 24) | (WINF - w)) == UNVIS;
}

// Level-synchronous BFS from `root` over the links with residual >= demand, labelling each
// reached vertex with its best (hops, width) to the root.  Stops after the level in which
// `stop` is discovered (stop < 0: runs to exhaustion).  Returns the level of `stop`, -1 if
// unreachable (stop < 0: the number of levels).  *S.tail = vertices reached (queue length).
template <class GR, class QT>
__device__ int warp_bfs(const GR& G, const Scratch2<QT>& S, int root, int demand, int stop,
                        unsigned long long* edges) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  if (lane == 0) {
    S.key[root] = 0u;
    S.queue[0] = (QT)root;
    *S.tail = 1;
  }
  __syncwarp();
  int head = 0, tail = 1, level = 0;
  unsigned long long cnt = 0;
  for (;;) {
    const unsigned nl = (unsigned)(level + 1) & 255u;
    bool found = false;
    for (int base = head; base < tail; base += 32) {
      const int i = base + lane;
      int v = -1, b = 0, e = 0;
      unsigned Wv = 0;
      if (i < tail) {
        v = (int)S.queue[i];
        Wv = width_of(((volatile unsigned*)S.key)[v]);
        b = G.begin(v);
        e = G.end(v);
        cnt += (unsigned)(e - b);
      }
      // light vertices: own lane
      if (e - b <= HEAVY) {
        for (int j = b; j < e; ++j) {
          const int2 a = G.edge(j);
          if (relax(S.key, a, Wv, nl, demand)) {
            S.queue[atomicAdd(S.tail, 1)] = (QT)a.x;
            found |= (a.x == stop);
          }
        }
      }
      // heavy vertices: the whole warp, one edge per lane
      unsigned heavy = __ballot_sync(FULL, e - b > HEAVY);
      while (heavy) {
        const int l = __ffs(heavy) - 1;
        heavy &= heavy - 1;
        const int hb = __shfl_sync(FULL, b, l), he = __shfl_sync(FULL, e, l);
        const unsigned hW = __shfl_sync(FULL, Wv, l);
        for (int j0 = hb; j0 < he; j0 += 32) {
          const int j = j0 + lane;
          bool nw = false;
          int2 a = make_int2(-1, 0);
          if (j < he) {
            a = G.edge(j);
            nw = relax(S.key, a, hW, nl, demand);
          }
          const unsigned m = __ballot_sync(FULL, nw);
          if (m) {
            int at = 0;
            if (lane == 0) at = atomicAdd(S.tail, __popc(m));
            at = __shfl_sync(FULL, at, 0);
            if (nw) {
              S.queue[at + __popc(m & lt)] = (QT)a.x;
              found |= (a.x == stop);
            }
          }
        }
      }
    }
    __syncwarp();
    const int nt = *(volatile int*)S.tail;
    head = tail;
    tail = nt;
    ++level;
    if (__any_sync(FULL, found)) break;
    if (head == tail) {
      level = stop < 0 ? level - 1 : -1;
      break;
    }
  }
  for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(FULL, cnt, o);
  if (lane == 0 && edges) *edges += cnt;
  return level;
}

template <class QT>
__device__ void warp_reset(const Scratch2<QT>& S, int tail) {
  for (int i = threadIdx.x & 31; i < tail; i += 32) S.key[(int)S.queue[i]] = UNVIS;
  __syncwarp();
}

// Walk src -> dst over the labels of a BFS from dst that stopped at level L = hops(src).
template <class GR, class QT>
__device__ void warp_walk(const GR& G, const Scratch2<QT>& S, int s, int d, int L, unsigned B, int* prow) {
  const int lane = threadIdx.x & 31;
  int v = s;
  if (lane == 0) prow[0] = s;
  for (int step = 1; step <= L; ++step) {
    const unsigned want = (unsigned)(L - step) & 255u;
    const int b = G.begin(v), e = G.end(v);
    int best = INT_MAX;
    for (int j = b + lane; j < e; j += 32) {
      const int2 a = G.edge(j);
      if (a.y < d) continue;
      const unsigned kw = ((volatile unsigned*)S.key)[a.x];
      if (kw == UNVIS || (kw >> 24) != want) continue;
      if (min((unsigned)a.y, width_of(kw)) < B) continue;
      best = min(best, a.x);
    }
    v = __reduce_min_sync(FULL, best);
    if (lane == 0) prow[step] = v;
  }
}

// Kernel prologue: the graph into shared memory (SMEM mode), per-warp scratch carved, keys
// set to UNVIS.  Shared layout (SMEM): off[V+1] | adj[2L] (u32) | per warp: key[V] | queue[V]
// (u16) | tail.  GLOBAL mode: per warp key[V] | queue[V] (int) | tail, in shared memory or
// in gscratch.
template <bool SM>
struct Setup;

template <>
struct Setup<true> {
  using QT = uint16_t;
  using GR = SmemGraph;
  __device__ static void run(const GraphDev& G, unsigned char* smem, unsigned*, int, GR* gr, Scratch2<QT>* S) {
    int* off = reinterpret_cast<int*>(smem);
    unsigned* adj = reinterpret_cast<unsigned*>(off + G.V + 1);
    const int n2 = G.n_adj;
    for (int i = threadIdx.x; i <= G.V; i += blockDim.x) off[i] = __ldg(G.off + i);
    for (int i = threadIdx.x; i < n2; i += blockDim.x) adj[i] = __ldg(G.adj16 + i);
    unsigned char* wb = reinterpret_cast<unsigned char*>(adj + n2);
    const size_t per = path_warp_bytes(G.V, true);
    wb += (size_t)(threadIdx.x >> 5) * per;
    S->key = reinterpret_cast<unsigned*>(wb);
    S->queue = reinterpret_cast<uint16_t*>(wb + 4 * (size_t)G.V);
    S->tail = reinterpret_cast<int*>(wb + per - 4);
    for (int i = threadIdx.x & 31; i < G.V; i += 32) S->key[i] = UNVIS;
    gr->off = off;
    gr->adj = adj;
    __syncthreads();
  }
};

template <>
struct Setup<false> {
  using QT = int;
  using GR = GlobalGraph;
  __device__ static void run(const GraphDev& G, unsigned char* smem, unsigned* gscratch, int warps, GR* gr,
                             Scratch2<QT>* S) {
    const size_t per = path_warp_bytes(G.V, false);
    const int w = threadIdx.x >> 5;
    unsigned char* wb = gscratch ? reinterpret_cast<unsigned char*>(gscratch) + ((size_t)blockIdx.x * warps + w) * per
                                 : smem + (size_t)w * per;
    S->key = reinterpret_cast<unsigned*>(wb);
    S->queue = reinterpret_cast<int*>(wb + 4 * (size_t)G.V);
    S->tail = reinterpret_cast<int*>(wb + per - 4);
    for (int i = threadIdx.x & 31; i < G.V; i += 32) S->key[i] = UNVIS;
    gr->off = G.off;
    gr->adj = G.adj;
    __syncwarp();
  }
};

// Writes the answer of query q from the labels of a BFS from dst (level L of s, width B):
// bottleneck, hops and (warp-cooperative walk) the path row.
template <class GR, class QT>
__device__ void answer(const GR& gr, const Scratch2<QT>& S, int q, int s, int d, int L, unsigned B, int* bn,
                       int* hops, int* path, int max_hops) {
  const int lane = threadIdx.x & 31;
  if (lane == 0) {
    bn[q] = L < 0 ? -1 : (int)B;
    hops[q] = L;
  }
  if (path) {
    int* prow = path + (size_t)q * (max_hops + 1);
    if (L < 0 || L > max_hops) {
      for (int i = lane; i <= max_hops; i += 32) prow[i] = -1;
    } else {
      warp_walk(gr, S, s, d, L, B, prow);
      for (int i = L + 1 + lane; i <= max_hops; i += 32) prow[i] = -1;
    }
  }
}

// One warp per (src, dst, demand) query (every query, or the queries idx[0 .. *n_idx) the
// grouped pass deferred).  Outputs: bn (bottleneck, -1 infeasible), hops (-1 infeasible, -2
// invalid query), path rows of max_hops + 1 vertices (-1 padded; all -1 when hops >
// max_hops or infeasible).
template <bool SM>
__global__ void __launch_bounds__(512) k_paths(GraphDev G, int nq, const int* __restrict__ src,
                                               const int* __restrict__ dst, const int* __restrict__ demand,
                                               int* bn, int* hops, int* path, int max_hops, const int* idx,
                                               const int* n_idx, unsigned* gscratch, int warps,
                                               unsigned long long* stats) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int n = n_idx ? *n_idx : nq;
  if (blockIdx.x * warps >= n) return;
  typename Setup<SM>::GR gr;
  Scratch2<typename Setup<SM>::QT> S;
  Setup<SM>::run(G, smem, gscratch, warps, &gr, &S);
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * warps + (threadIdx.x >> 5);
  const int nw = gridDim.x * warps;
  unsigned long long edges = 0, invalid = 0, runs = 0;
  for (int i = gw; i < n; i += nw) {
    const int q = idx ? idx[i] : i;
    const int s = __ldg(src + q), t = __ldg(dst + q), d = __ldg(demand + q);
    if (s < 0 || s >= G.V || t < 0 || t >= G.V || s == t || d < 0) {
      if (lane == 0) {
        bn[q] = -1;
        ++invalid;
      }
      answer(gr, S, q, s, d, -1, 0u, bn, hops, path, max_hops);
      if (lane == 0) hops[q] = -2;
      continue;
    }
    const int L = warp_bfs(gr, S, t, d, s, &edges);
    ++runs;
    const int tail = *(volatile int*)S.tail;
    const unsigned B = L < 0 ? 0u : width_of(((volatile unsigned*)S.key)[s]);
    answer(gr, S, q, s, d, L, B, bn, hops, path, max_hops);
    warp_reset(S, tail);
  }
  if (lane == 0) {
    if (edges) atomicAdd(stats + ST_EDGES, edges);
    if (invalid) atomicAdd(stats + ST_INVALID, invalid);
    if (runs) atomicAdd(stats + ST_BFS, runs);
  }
}

// ---- queries grouped by destination ---------------------------------------------------
// Exactness: let d0 be the smallest demand among the queries to t and label
// every vertex by a BFS from t over G_{d0} = {links with residual >= d0}.  For a query
// (s, t, d >= d0) whose label width W(s) >= d, the optimal paths of G_{d0} have bottleneck
// W(s) >= d, so they lie in G_d ⊆ G_{d0}: hop count, bottleneck and the set of optimal paths
// (hence the lexicographically smallest one) are those of G_d.  An unreachable s is
// unreachable in G_d too.  Only queries with W(s) < d need their own BFS (deferred).
// Layout of the group workspace (ints): cnt[V] | dmin[V] | start[V+1] | fill[V] | groups[V]
//   | ctr[4] (ngroups, next group, n deferred, spare) | order[nq] | deferred[nq].

__global__ void k_pg_init(int V, int* cnt, int* dmin, int* fill, int* ctr) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < V; i += gridDim.x * blockDim.x) {
    cnt[i] = 0;
    dmin[i] = INT_MAX;
    fill[i] = 0;
  }
  if (blockIdx.x == 0 && threadIdx.x < 4) ctr[threadIdx.x] = 0;
}

// count queries per destination and the smallest demand; invalid queries answered here
__global__ void k_pg_count(GraphDev G, int nq, const int* __restrict__ src, const int* __restrict__ dst,
                           const int* __restrict__ demand, int* cnt, int* dmin, int* bn, int* hops, int* path,
                           int max_hops, unsigned long long* stats) {
  unsigned long long invalid = 0;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += gridDim.x * blockDim.x) {
    const int s = __ldg(src + q), t = __ldg(dst + q), d = __ldg(demand + q);
    if (s < 0 || s >= G.V || t < 0 || t >= G.V || s == t || d < 0) {
      bn[q] = -1;
      hops[q] = -2;
      if (path)
        for (int i = 0; i <= max_hops; ++i) path[(size_t)q * (max_hops + 1) + i] = -1;
      ++invalid;
      continue;
    }
    atomicAdd(cnt + t, 1);
    atomicMin(dmin + t, d);
  }
  if (invalid) atomicAdd(stats + ST_INVALID, invalid);
}

// exclusive scan of cnt -> start, and the list of non-empty groups (one CTA)
__global__ void __launch_bounds__(1024) k_pg_scan(int V, const int* cnt, int* start, int* groups, int* ctr) {
  __shared__ int wsum[32], wsum2[32];
  __shared__ int carry_s, gcarry_s;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    carry_s = 0;
    gcarry_s = 0;
  }
  __syncthreads();
  for (int base = 0; base < V; base += 1024) {
    const int i = base + threadIdx.x;
    const int c = i < V ? cnt[i] : 0;
    const int ne = c > 0;
    int x = c, y = ne;
    for (int o = 1; o < 32; o <<= 1) {
      const int xo = __shfl_up_sync(FULL, x, o), yo = __shfl_up_sync(FULL, y, o);
      if (lane >= o) {
        x += xo;
        y += yo;
      }
    }
    if (lane == 31) {
      wsum[w] = x;
      wsum2[w] = y;
    }
    __syncthreads();
    if (w == 0) {
      int a = wsum[lane], b = wsum2[lane];
      for (int o = 1; o < 32; o <<= 1) {
        const int ao = __shfl_up_sync(FULL, a, o), bo = __shfl_up_sync(FULL, b, o);
        if (lane >= o) {
          a += ao;
          b += bo;
        }
      }
      wsum[lane] = a;
      wsum2[lane] = b;
    }
    __syncthreads();
    const int xpre = (w ? wsum[w - 1] : 0) + x - c + carry_s;
    const int ypre = (w ? wsum2[w - 1] : 0) + y - ne + gcarry_s;
    if (i < V) {
      start[i] = xpre;
      if (ne) groups[ypre] = i;
    }
    __syncthreads();
    if (threadIdx.x == 1023) {
      carry_s = xpre + c;
      gcarry_s = ypre + ne;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    start[V] = carry_s;
    ctr[0] = gcarry_s;
  }
}

__global__ void k_pg_scatter(GraphDev G, int nq, const int* __restrict__ src, const int* __restrict__ dst,
                             const int* __restrict__ demand, const int* start, int* fill, int* order) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += gridDim.x * blockDim.x) {
    const int s = __ldg(src + q), t = __ldg(dst + q), d = __ldg(demand + q);
    if (s < 0 || s >= G.V || t < 0 || t >= G.V || s == t || d < 0) continue;
    order[start[t] + atomicAdd(fill + t, 1)] = q;
  }
}

// One warp per destination group (taken from a work counter): one BFS from t over
// G_{dmin[t]} to exhaustion, then every query of the group answered from the labels by
// one lane (label lookup, then the walk to t: per hop the smallest-id neighbour one level
// closer that keeps the bottleneck), or deferred when W(s) < d (or when the BFS is deeper
// than the 8-bit level field).
template <bool SM>
__global__ void __launch_bounds__(512) k_paths_grouped(GraphDev G, const int* __restrict__ src,
                                                       const int* __restrict__ demand, const int* dmin,
                                                       const int* start, const int* groups, const int* order,
                                                       int* ctr, int* deferred, int* bn, int* hops, int* path,
                                                       int max_hops, unsigned* gscratch, int warps,
                                                       unsigned long long* stats) {
  extern __shared__ __align__(16) unsigned char smem[];
  typename Setup<SM>::GR gr;
  Scratch2<typename Setup<SM>::QT> S;
  Setup<SM>::run(G, smem, gscratch, warps, &gr, &S);
  const int lane = threadIdx.x & 31;
  const int ngroups = ctr[0];
  unsigned long long edges = 0, runs = 0;
  for (;;) {
    int gi = 0;
    if (lane == 0) gi = atomicAdd(ctr + 1, 1);
    gi = __shfl_sync(FULL, gi, 0);
    if (gi >= ngroups) break;
    const int t = groups[gi];
    const int d0 = dmin[t];
    const int depth = warp_bfs(gr, S, t, d0, -1, &edges);
    ++runs;
    const int tail = *(volatile int*)S.tail;
    const bool exact = depth <= 255;
    // the group's queries, one per lane: label lookup and a lane-serial walk
    for (int i = start[t] + lane; i < start[t + 1]; i += 32) {
      const int q = order[i];
      const int s = __ldg(src + q), d = __ldg(demand + q);
      const unsigned ks = ((volatile unsigned*)S.key)[s];
      const unsigned B = width_of(ks);
      if (!exact || (ks != UNVIS && B < (unsigned)d)) {
        deferred[atomicAdd(ctr + 2, 1)] = q;
        continue;
      }
      const int L = ks == UNVIS ? -1 : (int)(ks >> 24);
      bn[q] = L < 0 ? -1 : (int)B;
      hops[q] = L;
      if (path) {
        int* prow = path + (size_t)q * (max_hops + 1);
        int at = 0;
        if (L >= 0 && L <= max_hops) {
          int v = s;
          prow[at++] = v;
          for (int step = 1; step <= L; ++step) {
            const unsigned want = (unsigned)(L - step) & 255u;
            int best = INT_MAX;
            for (int j = gr.begin(v), e = gr.end(v); j < e; ++j) {
              const int2 a = gr.edge(j);
              if (a.y < d0 || a.x >= best) continue;
              const unsigned kw = ((volatile unsigned*)S.key)[a.x];
              if (kw == UNVIS || (kw >> 24) != want || min((unsigned)a.y, width_of(kw)) < B) continue;
              best = a.x;
            }
            v = best;
            prow[at++] = v;
          }
        }
        for (; at <= max_hops; ++at) prow[at] = -1;
      }
    }
    __syncwarp();
    warp_reset(S, tail);
  }
  if (lane == 0) {
    if (edges) atomicAdd(stats + ST_EDGES, edges);
    if (runs) atomicAdd(stats + ST_BFS, runs);
  }
}

// One warp per server u: BFS from u with every link usable (demand 0) to exhaustion, then
// out[u] = sum over the reached servers v != u of their widest-shortest bottleneck.
template <bool SM>
__global__ void __launch_bounds__(512) k_logical_bw(GraphDev G, long long* out, unsigned* gscratch, int warps,
                                                    unsigned long long* stats) {
  extern __shared__ __align__(16) unsigned char smem[];
  typename Setup<SM>::GR gr;
  Scratch2<typename Setup<SM>::QT> S;
  Setup<SM>::run(G, smem, gscratch, warps, &gr, &S);
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * warps + (threadIdx.x >> 5);
  const int nw = gridDim.x * warps;
  unsigned long long edges = 0;
  for (int u = gw; u < G.ns; u += nw) {
    warp_bfs(gr, S, u, 0, -1, &edges);
    const int tail = *(volatile int*)S.tail;
    long long s = 0;
    for (int i = 1 + lane; i < tail; i += 32) {
      const int v = (int)S.queue[i];
      if (v < G.ns) s += width_of(((volatile unsigned*)S.key)[v]);
    }
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
    if (lane == 0) out[u] = s;
    warp_reset(S, tail);
  }
  if (lane == 0 && edges) atomicAdd(stats + ST_EDGES, edges);
}

// ---- CTA-cooperative grouped kernel (shared-memory layout) ------------------------------
// One destination group per CTA at a time (work counter), all warps on its BFS: a frontier
// of a fat-tree level is hundreds of vertices, so 8 warps share it; per-CTA scratch is one
// key[V] + queue[V], so 3 CTAs (24 warps) fit an SM beside the graph copy, against 11 warps
// of private per-warp scratch, and 2000 groups spread over 444 CTAs instead of 1628 warps
// (the per-warp kernel ran 7.2 of 11 warps active: one or two groups per warp).
template <class GR, class QT>
__device__ int cta_bfs(const GR& G, unsigned* key, QT* queue, int* tailp, int root, int demand,
                       unsigned long long* edges) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, NW = blockDim.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  if (threadIdx.x == 0) {
    key[root] = 0u;
    queue[0] = (QT)root;
    *tailp = 1;
  }
  __syncthreads();
  int head = 0, tail = 1, level = 0;
  unsigned long long cnt = 0;
  for (;;) {
    const unsigned nl = (unsigned)(level + 1) & 255u;
    for (int base = head + warp * 32; base < tail; base += NW * 32) {
      const int i = base + lane;
      int b = 0, e = 0;
      unsigned Wv = 0;
      if (i < tail) {
        const int v = (int)queue[i];
        Wv = width_of(((volatile unsigned*)key)[v]);
        b = G.begin(v);
        e = G.end(v);
        cnt += (unsigned)(e - b);
      }
      if (e - b <= HEAVY) {
        for (int j = b; j < e; ++j) {
          const int2 a = G.edge(j);
          if (relax(key, a, Wv, nl, demand)) queue[atomicAdd(tailp, 1)] = (QT)a.x;
        }
      }
      unsigned heavy = __ballot_sync(FULL, e - b > HEAVY);
      while (heavy) {
        const int l = __ffs(heavy) - 1;
        heavy &= heavy - 1;
        const int hb = __shfl_sync(FULL, b, l), he = __shfl_sync(FULL, e, l);
        const unsigned hW = __shfl_sync(FULL, Wv, l);
        for (int j0 = hb; j0 < he; j0 += 32) {
          const int j = j0 + lane;
          bool nw = false;
          int2 a = make_int2(-1, 0);
          if (j < he) {
            a = G.edge(j);
            nw = relax(key, a, hW, nl, demand);
          }
          const unsigned m = __ballot_sync(FULL, nw);
          if (m) {
            int at = 0;
            if (lane == 0) at = atomicAdd(tailp, __popc(m));
            at = __shfl_sync(FULL, at, 0);
            if (nw) queue[at + __popc(m & lt)] = (QT)a.x;
          }
        }
      }
    }
    __syncthreads();
    const int nt = *(volatile int*)tailp;
    head = tail;
    tail = nt;
    ++level;
    __syncthreads();  // every thread has read the tail before the next level appends
    if (head == tail) {
      --level;
      break;
    }
  }
  for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(FULL, cnt, o);
  if (lane == 0 && edges) *edges += cnt;
  return level;
}

__global__ void __launch_bounds__(256) k_paths_grouped_cta(GraphDev G, const int* __restrict__ src,
                                                           const int* __restrict__ demand, const int* dmin,
                                                           const int* start, const int* groups, const int* order,
                                                           int* ctr, int* deferred, int* bn, int* hops, int* path,
                                                           int max_hops, unsigned long long* stats) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int gi_s, tail_s;
  int* off = reinterpret_cast<int*>(smem);
  unsigned* adj = reinterpret_cast<unsigned*>(off + G.V + 1);
  for (int i = threadIdx.x; i <= G.V; i += blockDim.x) off[i] = __ldg(G.off + i);
  for (int i = threadIdx.x; i < G.n_adj; i += blockDim.x) adj[i] = __ldg(G.adj16 + i);
  unsigned* key = reinterpret_cast<unsigned*>(
      reinterpret_cast<unsigned char*>(smem) + ((4 * ((size_t)G.V + 1) + 4 * (size_t)G.n_adj + 15) & ~(size_t)15));
  uint16_t* queue = reinterpret_cast<uint16_t*>(key + G.V);
  for (int i = threadIdx.x; i < G.V; i += blockDim.x) key[i] = UNVIS;
  SmemGraph gr;
  gr.off = off;
  gr.adj = adj;
  __syncthreads();
  const int ngroups = ctr[0];
  unsigned long long edges = 0, runs = 0;
  for (;;) {
    if (threadIdx.x == 0) gi_s = atomicAdd(ctr + 1, 1);
    __syncthreads();
    const int gi = gi_s;
    if (gi >= ngroups) break;
    const int t = groups[gi];
    const int d0 = dmin[t];
    const int depth = cta_bfs(gr, key, queue, &tail_s, t, d0, &edges);
    ++runs;
    const int tail = tail_s;
    const bool exact = depth <= 255;
    for (int i = start[t] + threadIdx.x; i < start[t + 1]; i += blockDim.x) {
      const int q = order[i];
      const int s = __ldg(src + q), d = __ldg(demand + q);
      const unsigned ks = ((volatile unsigned*)key)[s];
      const unsigned B = width_of(ks);
      if (!exact || (ks != UNVIS && B < (unsigned)d)) {
        deferred[atomicAdd(ctr + 2, 1)] = q;
        continue;
      }
      const int L = ks == UNVIS ? -1 : (int)(ks >> 24);
      bn[q] = L < 0 ? -1 : (int)B;
      hops[q] = L;
      if (path) {
        int* prow = path + (size_t)q * (max_hops + 1);
        int at = 0;
        if (L >= 0 && L <= max_hops) {
          int v = s;
          prow[at++] = v;
          for (int step = 1; step <= L; ++step) {
            const unsigned want = (unsigned)(L - step) & 255u;
            int best = INT_MAX;
            for (int j = gr.begin(v), e = gr.end(v); j < e; ++j) {
              const int2 a = gr.edge(j);
              if (a.y < d0 || a.x >= best) continue;
              const unsigned kw = ((volatile unsigned*)key)[a.x];
              if (kw == UNVIS || (kw >> 24) != want || min((unsigned)a.y, width_of(kw)) < B) continue;
              best = a.x;
            }
            v = best;
            prow[at++] = v;
          }
        }
        for (; at <= max_hops; ++at) prow[at] = -1;
      }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < tail; i += blockDim.x) key[(int)queue[i]] = UNVIS;
    __syncthreads();
  }
  if ((threadIdx.x & 31) == 0 && edges) atomicAdd(stats + ST_EDGES, edges);
  if (threadIdx.x == 0 && runs) atomicAdd(stats + ST_BFS, runs);
}

// Logical bandwidth with the CTA-cooperative BFS (shared-memory layout): a CTA per server u.
__global__ void __launch_bounds__(256) k_logical_bw_cta(GraphDev G, long long* out, unsigned long long* stats) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int tail_s;
  __shared__ long long part[8];
  int* off = reinterpret_cast<int*>(smem);
  unsigned* adj = reinterpret_cast<unsigned*>(off + G.V + 1);
  for (int i = threadIdx.x; i <= G.V; i += blockDim.x) off[i] = __ldg(G.off + i);
  for (int i = threadIdx.x; i < G.n_adj; i += blockDim.x) adj[i] = __ldg(G.adj16 + i);
  unsigned* key = reinterpret_cast<unsigned*>(
      reinterpret_cast<unsigned char*>(smem) + ((4 * ((size_t)G.V + 1) + 4 * (size_t)G.n_adj + 15) & ~(size_t)15));
  uint16_t* queue = reinterpret_cast<uint16_t*>(key + G.V);
  for (int i = threadIdx.x; i < G.V; i += blockDim.x) key[i] = UNVIS;
  SmemGraph gr;
  gr.off = off;
  gr.adj = adj;
  __syncthreads();
  unsigned long long edges = 0;
  for (int u = blockIdx.x; u < G.ns; u += gridDim.x) {
    cta_bfs(gr, key, queue, &tail_s, u, 0, &edges);
    const int tail = tail_s;
    long long sum = 0;
    for (int i = 1 + threadIdx.x; i < tail; i += blockDim.x) {
      const int v = (int)queue[i];
      if (v < G.ns) sum += width_of(((volatile unsigned*)key)[v]);
    }
    for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(FULL, sum, o);
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = sum;
    __syncthreads();
    if (threadIdx.x == 0) {
      long long t = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += part[w];
      out[u] = t;
    }
    for (int i = threadIdx.x; i < tail; i += blockDim.x) key[(int)queue[i]] = UNVIS;
    __syncthreads();
  }
  if ((threadIdx.x & 31) == 0 && edges) atomicAdd(stats + ST_EDGES, edges);
}

template <class K>
int occupancy(K kernel, int threads, size_t smem) {
  int blocks = 0;
  if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kernel, threads, smem) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return blocks;
}

}  // namespace

__host__ __device__ size_t path_warp_bytes(int V, bool smem_mode) {
  // key[V] u32 | queue[V] (u16 in SMEM mode, int otherwise) | tail, 16-byte aligned
  const size_t b = 4 * (size_t)V + (smem_mode ? 2 : 4) * (size_t)V + 4;
  return (b + 15) & ~(size_t)15;
}

PathLaunch path_launch_config(const GraphDev& G, int num_sms) {
  constexpr size_t SMAX = 227 * 1024;
  PathLaunch c{};
  if (G.adj16) {  // SMEM: graph + at least 4 warps of scratch on-chip
    const size_t gbytes = ((4 * ((size_t)G.V + 1) + 4 * (size_t)G.n_adj) + 15) & ~(size_t)15;
    const size_t per = path_warp_bytes(G.V, true);
    if (gbytes + 4 * per <= SMAX) {
      c.smem_graph = true;
      c.warps = (int)std::min<size_t>(16, (SMAX - gbytes) / per);
      c.dyn_smem = gbytes + per * c.warps;
      int blocks = occupancy(k_paths_grouped<true>, c.warps * 32, c.dyn_smem);
      c.grid = num_sms * std::max(1, blocks);
      // the CTA-cooperative grouped kernel: graph + one key[V] | queue[V] per CTA
      c.cta_smem = gbytes + ((6 * (size_t)G.V + 15) & ~(size_t)15);
      const int cb = occupancy(k_paths_grouped_cta, 256, c.cta_smem);
      c.cta_grid = cb > 0 ? num_sms * cb : 0;
      return c;
    }
  }
  const size_t per = path_warp_bytes(G.V, false);
  const int w = (int)std::min<size_t>(16, SMAX / per);
  if (w >= 2) {
    c.warps = w;
    c.dyn_smem = per * w;
    int blocks = occupancy(k_paths_grouped<false>, w * 32, c.dyn_smem);
    c.grid = num_sms * std::max(1, blocks);
  } else {
    c.warps = 16;
    c.dyn_smem = 0;
    c.grid = num_sms * 2;
    c.global_bytes = (size_t)c.grid * c.warps * per;
  }
  return c;
}

size_t path_group_ints(int V, int nq) { return 5 * (size_t)V + 1 + 4 + 2 * (size_t)nq; }

template <bool SM>
static cudaError_t launch_paths_t(const GraphDev& G, const PathLaunch& c, int nq, const int* src, const int* dst,
                                  const int* demand, int* bn, int* hops, int* path, int max_hops, int* ws,
                                  unsigned* gscratch, unsigned long long* stats, cudaStream_t st) {
  const int V = G.V;
  int* cnt = ws;
  int* dmin = cnt + V;
  int* start = dmin + V;
  int* fill = start + V + 1;
  int* groups = fill + V;
  int* ctr = groups + V;
  int* order = ctr + 4;
  int* deferred = order + nq;
  unsigned* gs = c.global_bytes ? gscratch : nullptr;
  cudaError_t e = cudaFuncSetAttribute(k_paths_grouped<SM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)c.dyn_smem);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_paths<SM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c.dyn_smem);
  if (e != cudaSuccess) return e;
  const int eg = std::min(1184, (std::max(nq, V) + 255) / 256);
  k_pg_init<<<std::min(1184, (V + 255) / 256), 256, 0, st>>>(V, cnt, dmin, fill, ctr);
  k_pg_count<<<eg, 256, 0, st>>>(G, nq, src, dst, demand, cnt, dmin, bn, hops, path, max_hops, stats);
  k_pg_scan<<<1, 1024, 0, st>>>(V, cnt, start, groups, ctr);
  k_pg_scatter<<<eg, 256, 0, st>>>(G, nq, src, dst, demand, start, fill, order);
  if (SM && c.cta_grid > 0) {
    e = cudaFuncSetAttribute(k_paths_grouped_cta, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c.cta_smem);
    if (e != cudaSuccess) return e;
    k_paths_grouped_cta<<<c.cta_grid, 256, c.cta_smem, st>>>(G, src, demand, dmin, start, groups, order, ctr,
                                                              deferred, bn, hops, path, max_hops, stats);
  } else
  k_paths_grouped<SM><<<c.grid, c.warps * 32, c.dyn_smem, st>>>(G, src, demand, dmin, start, groups, order, ctr,
                                                                deferred, bn, hops, path, max_hops, gs, c.warps,
                                                                stats);
  k_paths<SM><<<c.grid, c.warps * 32, c.dyn_smem, st>>>(G, nq, src, dst, demand, bn, hops, path, max_hops,
                                                        deferred, ctr + 2, gs, c.warps, stats);
  return cudaGetLastError();
}

cudaError_t launch_paths(const GraphDev& G, const PathLaunch& c, int nq, const int* src, const int* dst,
                         const int* demand, int* bn, int* hops, int* path, int max_hops, int* ws,
                         unsigned* gscratch, unsigned long long* stats, cudaStream_t st) {
  if (nq <= 0) return cudaSuccess;
  return c.smem_graph ? launch_paths_t<true>(G, c, nq, src, dst, demand, bn, hops, path, max_hops, ws, gscratch,
                                             stats, st)
                      : launch_paths_t<false>(G, c, nq, src, dst, demand, bn, hops, path, max_hops, ws, gscratch,
                                              stats, st);
}

cudaError_t launch_logical_bw(const GraphDev& G, const PathLaunch& c, long long* out, unsigned* gscratch,
                              unsigned long long* stats, cudaStream_t st) {
  if (G.ns <= 0) return cudaSuccess;
  const int grid = std::min(c.grid, (G.ns + c.warps - 1) / c.warps);
  unsigned* gs = c.global_bytes ? gscratch : nullptr;
  if (c.smem_graph && c.cta_grid > 0) {
    cudaError_t e = cudaFuncSetAttribute(k_logical_bw_cta, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)c.cta_smem);
    if (e != cudaSuccess) return e;
    k_logical_bw_cta<<<std::min(c.cta_grid, G.ns), 256, c.cta_smem, st>>>(G, out, stats);
  } else if (c.smem_graph) {
    cudaError_t e = cudaFuncSetAttribute(k_logical_bw<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)c.dyn_smem);
    if (e != cudaSuccess) return e;
    k_logical_bw<true><<<grid, c.warps * 32, c.dyn_smem, st>>>(G, out, gs, c.warps, stats);
  } else {
    cudaError_t e = cudaFuncSetAttribute(k_logical_bw<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)c.dyn_smem);
    if (e != cudaSuccess) return e;
    k_logical_bw<false><<<grid, c.warps * 32, c.dyn_smem, st>>>(G, out, gs, c.warps, stats);
  }
  return cudaGetLastError();
}

}  // namespace nacs
