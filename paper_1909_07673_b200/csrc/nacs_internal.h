// nacs_internal.h — types shared by the host API (nacs_api.cu) and the kernels
// (nacs_kernels.cu) of libnacs.  Not part of the public ABI (include/nacs.h).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace nacs {

constexpr int MAXC = 128;   // NACS_MAX_CONTAINERS: containers (and pods) per request
constexpr int MAXV = 512;   // NACS_MAX_VLINKS: virtual links per request
constexpr int MAXF = 128;   // flows per pod step (one per distinct peer server, <= pods)
constexpr int MAXK = 64;    // NACS_MAX_K
constexpr int MAXW = 32;    // warps per CTA
// undo-log entries one request can need: 3 per pod + 6 per flow + 2 per container
// (top-up) + 6 per vlink (top-up); every vlink belongs to at most one flow.
constexpr int ULOG_CAP = 3 * MAXC + 6 * MAXV + 2 * MAXC + 6 * MAXV + 64;

// Fat-tree geometry (include/nacs.h).  Device state layout, int32 words:
//   cpu[n] | ram[n] | act[n] | links[L] = access[n] | edge-agg[E*h] | agg-core[k*h*h]
// so the criteria table (cpu, ram, act, acc) is the first 4n words, structure-of-arrays.
struct Geo {
  int k, h, n, E, L;
  int cpu_cap, ram_cap, link_cap;
  unsigned magic_h;  // ceil(2^32 / h): x / h == __umulhi(x, magic_h) for x < 2^24; 0 for h = 1 (div_h)
  __host__ __device__ int words() const { return 3 * n + L; }
};

struct Opt {
  int method;        // 0 AHP, 1 TOPSIS
  double wd[4];      // weights W
  int ahp_rule;      // 0 literal, 1 shifted
  int l1_mode;       // 0 pairwise on W, 1 L1 = W
  int path_filter;   // 1 filter on path bandwidth, 0 CPU/RAM only
  int exact64;       // decide every argmax in FP64
  int rank_once;     // R25: rank once per request (the first pod step's order), pods walk it
  int bw_logical;    // R2 alternative: logical-bandwidth criterion (rank calls only)
};

struct ReqsDev {
  int n;
  const int *coff, *cpu_min, *cpu_max, *ram_min, *ram_max, *pod_of;
  const int *voff, *src, *dst, *bw_min, *bw_max;
};

struct OutDev {
  int *status, *server, *cpu_a, *ram_a, *bw_a, *path;
};

struct QueryDev {
  int dc, dr, nflow, nex;
  const int *fv, *fD, *ex;  // device arrays
  uint8_t *mask;            // [n] or null
  float *scores;            // [n] or null
  int *best;                // [1]
  const int* crit;          // [4n] criteria rows with the logical bandwidth (bw_criterion = 1), or null
};

enum {
  ST_POD_STEPS = 0,
  ST_RETRIES = 1,
  ST_FP64 = 2,
  ST_INVALID = 3,
  ST_FEAS = 4,
  ST_PAIRS = 5,
  ST_SCAN_A = 6,  // slots read by pass A / pass B of the TOPSIS warp kernel
  ST_SCAN_B = 7,
  ST_EDGES = 8,   // general-topology path kernels: adjacency entries scanned
  ST_BFS = 9,     // ... and BFS traversals run
  ST_N = 10
};
// Workspace of the warp kernel's chunk layout (k_warp_layout), int words:
// [0..3] thresholds of the low region | criteria tiles [4 npad] | chunk table [16 nch] | inv[n]
constexpr int LAY_PST = 4;

// Request validation shared by the host path and the kernels (reading R24).
// Returns 0 if valid, else a bitmask: 1 size limit, 2 demands, 4 min>max, 8 pod ids,
// 16 vlink endpoints, 32 vlink bandwidth.
__host__ __device__ inline int validate_request(int nC, int nV, const int* cpu_min, const int* cpu_max,
                                                const int* ram_min, const int* ram_max, const int* pod_of,
                                                const int* src, const int* dst, const int* bw_min,
                                                const int* bw_max) {
  if (nC <= 0 || nC > MAXC || nV < 0 || nV > MAXV) return 1;
  int bad = 0;
  unsigned used[MAXC / 32] = {0, 0, 0, 0};
  int maxp = -1;
  for (int i = 0; i < nC; ++i) {
    if (cpu_min[i] <= 0 || ram_min[i] <= 0) bad |= 2;
    if (cpu_min[i] > cpu_max[i] || ram_min[i] > ram_max[i]) bad |= 4;
    int p = pod_of[i];
    if (p < 0 || p >= nC) { bad |= 8; continue; }
    used[p >> 5] |= 1u << (p & 31);
    if (p > maxp) maxp = p;
  }
  for (int p = 0; p <= maxp; ++p)
    if (!((used[p >> 5] >> (p & 31)) & 1u)) bad |= 8;
  for (int e = 0; e < nV; ++e) {
    if (src[e] < 0 || src[e] >= nC || dst[e] < 0 || dst[e] >= nC || src[e] == dst[e]) bad |= 16;
    if (bw_min[e] <= 0 || bw_min[e] > bw_max[e]) bad |= 32;
  }
  return bad;
}

// Device pointers of the server-sharded engine (nacs_kernels.cu, k_sh_*).
struct Scratch;
// warps per criterion of the grid engine's between-passes kernels (k_ahp_mid_a / _b)
constexpr int AHP_MID_WARPS = 128;

struct ShardDev {
  Scratch* gs;                 // per-request scratch (global memory)
  unsigned *maskw, *special, *edgebad;
  int2* ulog;
  int* ctl;                    // [0] phase, [1] pod
  unsigned long long* kx;      // [2 * world] top-2 keys per rank
  double* kxv;                 // [world] FP64 best value per rank
  int* kxi;                    // [world] FP64 best server per rank
  unsigned long long* stats;
  // AHP (sorted levels of every criterion at once, see nacs_kernels.cu)
  unsigned char* ahp_ws;       // ahp_carve region: presort, merge buffers, priorities
  float2 *lvmC, *lvwC;         // [4][n2] (value, multiplicity), (value, weight) per level
  double *paC, *pbC;           // [4][n2+2] prefix sums
  int* lvlC;                   // [4][n] level of each server
  float *wq, *l2q;             // [4][n2] pass-1 weights, L2 per level (allreduced)
  double *wq64, *l2q64;        // [4][n2] FP64 re-decision
  int* Kc;                     // [4] levels per criterion (0 = constant criterion)
  unsigned long long* facc;    // [16]: [0..10] the grid filter's statistics (k_sh_filter), [15] presort flag
  int* lvscr;                  // AHP: per-criterion level-extraction scratch, 4 x [5 (n2 + 1)] ints
  unsigned long long* kpart;   // AHP: per-CTA top-2 keys of k_ahp_pg, [2 * npart]
  int npart;                   // CTAs of k_ahp_pg
  double* midtot;              // AHP: [4][AHP_MID_WARPS][2] segment totals of the between-passes scans
};

// Launchers (nacs_kernels.cu).  Each returns the cudaError_t of the launch.
struct LaunchInfo {
  int grid, block;
  size_t dyn_smem;
};

// AHP workspaces (nacs_kernels.cu): bytes of the sorted-level arrays for n servers, and
// doubles of the FP64 re-decision workspace (per CTA)
size_t ahp_workspace_bytes(int n);
size_t ahp_workspace_doubles(int n);
// dynamic shared memory of the batch kernel, 0 if it does not fit
size_t batch_smem_bytes(const Geo& g, int method);
// AHP batch with the sorted-level workspace in global memory (per CTA: ahp_workspace_bytes(n),
// 16-byte aligned) because it does not fit in shared memory beside the snapshot
bool batch_ahp_global(const Geo& g, int method);
int batch_block_size(const Geo& g, int method);
cudaError_t batch_occupancy(const Geo& g, int method, int* blocks_per_sm);

cudaError_t launch_batch(const Geo& g, const Opt& o, const int* d_state, const ReqsDev& R, const OutDev& O,
                         int2* ulog, double* w64, unsigned char* ahp_g, int* next, unsigned long long* stats,
                         int grid, cudaStream_t s, const int* idx = nullptr, const int* n_idx = nullptr);
// warp-per-request TOPSIS batch kernel (nacs_warp.cu): warps per CTA (0 = does not fit)
int warp_kernel_warps(const Geo& g);
size_t warp_ulog_entries(int grid, int warps);
size_t warp_layout_ints(const Geo& g);
cudaError_t launch_batch_warp(const Geo& g, const Opt& o, const int* d_state, int* lay, const ReqsDev& R,
                              const OutDev& O, int4* ulog, int* next, int* order, int* deferred, int* n_deferred,
                              unsigned long long* stats, int grid, int warps, cudaStream_t st);
// sequential: one CTA, requests in order, in place on d_state
cudaError_t launch_sequential(const Geo& g, const Opt& o, int* d_state, const ReqsDev& R, const OutDev& O,
                              int2* ulog, float* ahp_ws, double* w64, unsigned long long* stats,
                              cudaStream_t s);
// sequential TOPSIS on one thread-block cluster of C CTAs (large n; 0 = not used)
int seq_cluster_size(const Geo& g);
cudaError_t launch_seq_cluster(const Geo& g, const Opt& o, int* d_state, const ReqsDev& R, const OutDev& O,
                               int2* ulog, unsigned long long* stats, unsigned long long* work, int C,
                               cudaStream_t st);
cudaError_t launch_rank(const Geo& g, const Opt& o, int* d_state, const QueryDev& q, float* ahp_ws,
                        double* w64, unsigned long long* stats, cudaStream_t s);
cudaError_t launch_validate(const ReqsDev& R, int* status, unsigned long long* stats, cudaStream_t s);
// Whole-GPU TOPSIS ranking of one pod step on B DC states (nacs_rank.cu): a thread-block
// cluster of rank_many_cluster(g) CTAs per state, a persistent grid of clusters.
struct RankManyArgs {
  Geo g;
  double wd[4];
  int path_filter, exact64;
  const int* states;       // [B] states of g.words() int32 words, `stride` words apart
  long long stride;
  int B;
  int dc, dr, nflow, nex;  // the pod query (shared by every state)
  const int *fv, *fD, *ex; // device arrays: flows sorted by server, excluded servers
  uint8_t* mask;           // [B][n] or null
  float* scores;           // [B][n] or null
  int* best;               // [B]: argmax, -1 none feasible, -2 a value out of range
  unsigned long long* stats;
  int slice;               // set by the launcher
};
int rank_many_cluster(const Geo& g);
cudaError_t launch_rank_many(const RankManyArgs& a, int num_sms, cudaStream_t st);
// R2's logical bandwidth criterion on the current fat-tree state: crit = cpu | ram | act | L(u)
// ([4n]); F: [E*E] scratch; *too_big = 1 if some L(u) >= 2^24 (not exact in FP32)
cudaError_t launch_logical_criteria(const Geo& g, const int* state, int* crit, int* F, int* too_big,
                                    cudaStream_t st);
size_t scratch_bytes();
cudaError_t launch_sh_begin(const Geo& g, const Opt& o, int* state, const ReqsDev& R, const OutDev& O, int r,
                            const ShardDev& d, cudaStream_t st);
cudaError_t launch_sh_prep(const Geo& g, const Opt& o, int* state, const ReqsDev& R, const OutDev& O, int r,
                           const ShardDev& d, cudaStream_t st);
cudaError_t launch_sh_score(const Geo& g, const Opt& o, int* state, int lo, int hi, int slot, const ShardDev& d,
                            cudaStream_t st);
cudaError_t launch_sh_decide(const Geo& g, const Opt& o, int* state, const ReqsDev& R, const OutDev& O, int r,
                             int world, const ShardDev& d, cudaStream_t st);
cudaError_t launch_sh_fp64(const Geo& g, const Opt& o, int* state, int lo, int hi, int slot, const ShardDev& d,
                           cudaStream_t st);
cudaError_t launch_sh_decide64(const Geo& g, const Opt& o, int* state, const ReqsDev& R, const OutDev& O, int r,
                               int world, const ShardDev& d, cudaStream_t st);
// AHP pod step over the grid and the ranks: passes over this process's share of level
// pairs (ranks q in [q0, q1) of world), then the 1-CTA middle / decide kernels.
cudaError_t launch_ahp_pass(int pass, bool fp64, const Geo& g, const Opt& o, int* state, int q0, int q1, int world,
                            const ShardDev& d, int num_sms, cudaStream_t st);
cudaError_t launch_ahp_mid(bool fp64, const Geo& g, const Opt& o, int* state, const ShardDev& d, cudaStream_t st);
cudaError_t launch_ahp_decide(bool fp64, const Geo& g, const Opt& o, int* state, const ReqsDev& R, const OutDev& O,
                              int r, const ShardDev& d, cudaStream_t st);
cudaError_t launch_presort_update(const Geo& g, const Opt& o, int* state, const ShardDev& d, cudaStream_t st);

// departures (nacs_release, nacs_simulate): idx = null releases every request of R with
// status 1, else the requests idx[0 .. n_idx); delta: g.words() int64 scratch; bad: 1 int
// (1 malformed placement, 2 a residual would exceed its capacity; nothing applied then)
cudaError_t launch_release(const Geo& g, int* state, const ReqsDev& R, const OutDev& P, const int* idx, int n_idx,
                           long long* delta, int* bad, cudaStream_t st);
// the discrete-event run on the device (k_simulate, one CTA, one launch)
struct SimDev {
  const int *order, *arrival, *duration;  // order: requests by arrival tick, then id
  int max_ticks, hol;
  int *start, *attempts;                  // [R]
  int* ticks;                             // [max_ticks][3]: active servers, active links, queue
  int *qbuf, *qtmp, *run;                 // [R] each: queue, next queue, departure-bucket links
  int* head;                              // [max_ticks] first request departing at each tick (-1)
  long long* totals;                      // [3]: events (ticks), attempts, accepted
};
cudaError_t launch_simulate(const Geo& g, const Opt& o, int* d_state, const ReqsDev& R, const OutDev& O,
                            int2* ulog, float* ahp_ws, double* w64, unsigned long long* stats, const SimDev& S,
                            cudaStream_t st);
// active servers and active links of the current state into out[0..1]
cudaError_t launch_tick_counts(const Geo& g, const int* state, int* out, cudaStream_t st);

// General-topology graph (nacs_load_graph, nacs_paths.cu): CSR adjacency of the undirected
// links, both directions; adj[j] = (neighbour, residual); adj16[j] = neighbour | residual << 16
// (only when V <= 65536 and every residual <= 65535, else null).
struct GraphDev {
  int V, ns;
  int n_adj;              // 2 * n_links
  const int* off;         // [V+1]
  const int2* adj;        // [n_adj]
  const unsigned* adj16;  // [n_adj] or null
};
struct PathLaunch {
  int grid, warps;
  bool smem_graph;       // graph + per-warp scratch in shared memory
  size_t dyn_smem;
  size_t global_bytes;   // per-warp scratch in global memory (grid * warps * path_warp_bytes) when V is too large
  int cta_grid;          // CTA-cooperative grouped kernel (shared-memory layout), 0 = not used
  size_t cta_smem;
};
__host__ __device__ size_t path_warp_bytes(int V, bool smem_mode);
PathLaunch path_launch_config(const GraphDev& G, int num_sms);
// queries grouped by destination (one BFS per destination) + per-query BFS for the deferred
// ones; ws: path_group_ints(V, nq) ints of device workspace
size_t path_group_ints(int V, int nq);
cudaError_t launch_paths(const GraphDev& G, const PathLaunch& c, int nq, const int* src, const int* dst,
                         const int* demand, int* bn, int* hops, int* path, int max_hops, int* ws,
                         unsigned* gscratch, unsigned long long* stats, cudaStream_t st);
cudaError_t launch_logical_bw(const GraphDev& G, const PathLaunch& c, long long* out, unsigned* gscratch,
                              unsigned long long* stats, cudaStream_t st);

}  // namespace nacs
