/* nacs.h — C ABI of libnacs: the per-pod server ranking and placement hot path of
 * arXiv 1909.07673, "Network-Aware Container Scheduling in Multi-Tenant Data Center"
 * (§V), running as hand-written sm_100a CUDA kernels.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n (paper section / equation named
 * beside it); readings R1-R24 are listed in DESIGN.md §3.
 *
 * Units (reading R5): every quantity is an int32 in fixed units — CPU in millicores,
 * RAM in MiB, bandwidth in Mbps.  Every capacity must be <= NACS_MAX_CAP so that all
 * residuals and differences are exact in FP32 on the device.
 *
 * Ownership: the caller owns every input and output array.  The library copies inputs
 * during the call and never retains caller pointers.  The context owns its device
 * buffers and releases them in nacs_destroy().
 *
 * Pointers: host pointers unless nacs_options.flags has NACS_DEVICE_PTRS, in which case
 * every array passed to that call is a device pointer on the context's device (for
 * example a torch tensor's data_ptr()).  With NACS_ASYNC the call is stream-ordered on
 * the context stream and returns without synchronising; the caller synchronises the
 * stream before reading outputs.  Without NACS_ASYNC every call is synchronous.
 *
 * Errors: calls return nacs_status.  Invalid parameters are errors (NACS_EINVAL);
 * nacs_last_error() lists every violation found.  On any error the context state is
 * unchanged.  A request that cannot be placed is not an error: its status is 0 and all
 * its mappings are -1.  A context is single-writer and not thread-safe.
 */
#ifndef NACS_H
#define NACS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct nacs_ctx nacs_ctx;

typedef enum {
  NACS_OK = 0,
  NACS_EINVAL = 1,   /* invalid argument (see nacs_last_error) */
  NACS_ENOMEM = 2,   /* device or pinned host allocation failed */
  NACS_ECUDA = 3,    /* a CUDA runtime call failed */
  NACS_ENCCL = 4,    /* reserved for the server-sharded mode */
  NACS_ENOTOPO = 5,  /* no topology loaded */
  NACS_ETOOBIG = 6   /* a size limit below is exceeded */
} nacs_status;

/* NACS_BF / NACS_WF: the container orchestrators' native baselines the paper compares
 * against, "BF (binpacking) and WF (spread)" with "a shortest-path search after the
 * allocation of servers" (§IV; T5 P:416-426; reading R27): the feasible server
 * (CPU/RAM filter; options.path_filter is ignored and taken as 0) of smallest (BF) or
 * largest (WF) mean residual fraction (cpu/cpu_cap + ram/ram_cap)/2, ties lowest index;
 * routing, R18 retries and the R19 top-up as for the heuristics.  Schedule calls only. */
typedef enum { NACS_AHP = 0, NACS_TOPSIS = 1, NACS_BF = 2, NACS_WF = 3 } nacs_method;

/* nacs_options.flags */
#define NACS_DEVICE_PTRS 1u  /* arrays are device pointers */
#define NACS_ASYNC 2u        /* stream-ordered, no synchronisation (implies no host-side validation) */
#define NACS_EXACT_FP64 4u   /* decide every argmax in FP64 (the FP32 pass still runs) */

/* Limits. */
#define NACS_MAX_CAP 8388607     /* 2^23 - 1: every value exact in FP32 */
#define NACS_MAX_K 64            /* fat-tree arity: h = k/2 <= 32 aggregation switches per pod */
#define NACS_MAX_CONTAINERS 128  /* containers (hence pods) per request */
#define NACS_MAX_VLINKS 512      /* virtual links per request */

/* G^s(N^s, E^s) as a k-ary fat-tree (§II-A; §IV-B1; Table 1).
 * n = k^3/4 servers, h = k/2, E = k^2/2 edge switches, L = 3k^3/4 physical links.
 * Server u hangs off edge switch u / h; edge switch e lies in pod e / h.
 * Canonical link order: access[n] (server u <-> its edge switch) |
 *   edge-agg[E][h] (edge e <-> aggregation switch a of its pod) |
 *   agg-core[k][h][h] (aggregation switch a of pod p <-> core switch (a, b)).
 * Links are undirected with one shared residual (§V-D).
 * All arrays are host pointers. */
typedef struct {
  int32_t k;                             /* even, 2 <= k <= NACS_MAX_K */
  int32_t cpu_cap, ram_cap, link_cap;    /* homogeneous capacities, 1..NACS_MAX_CAP */
  const int32_t *cpu_res, *ram_res;      /* [n] residual c^s_u[r] in [0, cap]; NULL = fresh */
  const uint8_t *active;                 /* [n] f_u in {0,1}; NULL = derived: res < cap (R22) */
  const int32_t *link_res;               /* [L] residual bw in [0, link_cap]; NULL = fresh */
} nacs_topology;

/* One pod step for nacs_rank_*: the pod's summed c^min and its flows to
 * already-placed peer pods (R17): flow f goes to server flow_server[f] with aggregate
 * bw^min demand flow_bw[f] > 0 (servers distinct).  excluded[] servers are never
 * feasible (R18 retries). */
typedef struct {
  int32_t cpu_demand, ram_demand;        /* > 0 */
  int32_t n_flows;                       /* 0..NACS_MAX_CONTAINERS */
  const int32_t *flow_server, *flow_bw;  /* [n_flows] */
  int32_t n_excluded;                    /* 0..n */
  const int32_t *excluded;               /* [n_excluded] */
} nacs_pod_query;

/* A batch of requests Req(N^c, E^c) in CSR form (§II-A; Table 1).
 * Request r owns containers container_off[r] .. container_off[r+1]-1 and virtual links
 * vlink_off[r] .. vlink_off[r+1]-1; vl_src / vl_dst are request-local container ids.
 * pod_of[i] is the request-local pod id of container i; the ids must be exactly
 * 0..P-1 and pods are placed in ascending id (R15). */
typedef struct {
  int32_t n_requests;
  const int32_t *container_off;                          /* [n_requests+1], starts at 0 */
  const int32_t *cpu_min, *cpu_max, *ram_min, *ram_max;  /* per container: 0 < min <= max */
  const int32_t *pod_of;                                 /* per container */
  const int32_t *vlink_off;                              /* [n_requests+1], starts at 0 */
  const int32_t *vl_src, *vl_dst, *bw_min, *bw_max;      /* per vlink: src != dst, 0 < min <= max */
} nacs_requests;

/* Outputs M_c, M_ec, c^a, bw^a (Table 2), caller-allocated, sized like
 * the request arrays.  status: 1 accepted, 0 rejected (no feasible server for a pod,
 * R20), -1 invalid request (device-pointer calls and host-pointer nacs_schedule_batch
 * calls, which validate on the host while the kernels run and then also return
 * NACS_EINVAL / NACS_ETOOBIG naming the first invalid requests; host-pointer
 * nacs_schedule_request calls validate first and return the error before any work).  A non-accepted request has all mappings -1 and all
 * allocations 0.  path_of_vlink: -1 intra-server; 0 same edge switch; 1+a via
 * aggregation switch a of the shared pod; 1+h+a*h+b via core switch (a,b). */
typedef struct {
  int32_t *status;               /* [n_requests] */
  int32_t *server_of_container;  /* [sum containers] */
  int32_t *cpu_alloc, *ram_alloc;/* [sum containers] c^a within [c^min, c^max] (R19) */
  int32_t *bw_alloc;             /* [sum vlinks] bw^a within [bw^min, bw^max] (R19) */
  int32_t *path_of_vlink;        /* [sum vlinks] */
} nacs_placements;

/* Method options.  weights: W over (CPU, RAM, Fragmentation, Bandwidth) (Table 4
 * P:319-330, R1), finite, >= 0, |sum - 1| <= 1e-6 (R24). */
typedef struct {
  nacs_method method;
  double weights[4];
  int32_t ahp_rule;     /* 0 literal cell d / 1/(-d) / 1 (R8, default); 1 shifted 1+d / 1/(1-d) / 1 */
  int32_t l1_mode;      /* 0 L1 = AHP pairwise priority of W (R10, default); 1 L1 = W */
  int32_t path_filter;  /* 1 filter on path bandwidth (R6, default); 0 CPU/RAM-only filter */
  uint32_t flags;       /* NACS_DEVICE_PTRS | NACS_ASYNC | NACS_EXACT_FP64 */
  int32_t rank_mode;    /* NACS_RANK_PER_POD (R15, default): re-rank at every pod step;
                         * NACS_RANK_ONCE (R25, "sorted on decreasing order"
                         * P:375): the request's first pod step ranks the servers once and every
                         * pod takes the first server of that order its own filter (R6) admits.
                         * Schedule calls only; not on server-sharded contexts (NACS_EINVAL). */
  int32_t bw_criterion; /* NACS_BW_ACCESS (R2, default): the Bandwidth criterion is the residual of
                         * the server's access link; NACS_BW_LOGICAL (R2's alternative, "the sum of
                         * all bandwidth capacity bw^s_uv with source on u"; SURVEY 8(f) row
                         * 4): the sum over servers v != u of the widest-shortest u-v bottleneck on
                         * the current state.  nacs_rank_* only (schedule calls: NACS_EINVAL; the
                         * table would change after every commit); NACS_ETOOBIG when some sum
                         * reaches 2^24 (not exact in FP32, R5: n x link_cap must stay below it,
                         * e.g. k <= 32 at 1 Gbps).  The feasibility filter keeps the access links. */
} nacs_options;

enum { NACS_RANK_PER_POD = 0, NACS_RANK_ONCE = 1 };
enum { NACS_BW_ACCESS = 0, NACS_BW_LOGICAL = 1 };

/* Counters of the last rank/schedule call (reading them synchronises the context stream). */
typedef struct {
  int64_t pod_steps;       /* rankings run (every pod step and every R18 retry) */
  int64_t servers_ranked;  /* pod_steps x n */
  int64_t retries;         /* R18 commit failures */
  int64_t fp64_decisions;  /* argmaxes decided by the FP64 near-tie rescore */
  int64_t invalid;         /* requests rejected as invalid on the device */
  int64_t feasible;        /* sum over pod steps of |F| (feasible servers) */
  int64_t ahp_pairs;       /* AHP: sum over pod steps and non-constant criteria of the unordered pairs
                            * of DISTINCT levels K(K-1)/2 (the sorted-level passes' reciprocal terms) */
  int64_t scanned_a;       /* TOPSIS batch fast path: server slots read by the filter/statistics pass */
  int64_t scanned_b;       /* ... and by the scoring pass (chunk-pruned; 0 for the other kernels) */
  int64_t edges_scanned;   /* general-topology calls: adjacency entries read by the BFS levels */
  int64_t bfs_runs;        /* ... and BFS traversals run (one per destination group + deferred queries) */
} nacs_stats;

/* Create a context on CUDA device `device`.  cuda_stream: the cudaStream_t all work of
 * the context is ordered on (NULL = the legacy default stream, as in the CUDA runtime). */
nacs_status nacs_create(nacs_ctx **out, int device, void *cuda_stream);

/* Create a context that takes part in server-sharded scheduling (one huge
 * topology over `world` ranks, one process per GPU): every rank loads the same topology
 * and calls nacs_schedule_request with the same requests; each rank scores its own block
 * of world-th of the servers and the ranks exchange their (score, index) top-2 keys per
 * pod step with ncclAllGather over NVLink; every rank applies the same commit, so the
 * replicated states stay identical.  nccl_unique_id: the 128-byte ncclUniqueId from
 * nacs_nccl_unique_id() on rank 0, broadcast by the caller (e.g. torch.distributed);
 * NULL with world > 1 = loopback: all `world` logical shards run on this device (testing).
 * TOPSIS: each rank scores its server block and the ranks allgather their top-2 keys; AHP:
 * the level pairs of both passes are split over the ranks (whole tiles, so any rank count
 * gives bit-identical sums) and the per-level weights and L2 are sum-allreduced.
 * After an error inside a sharded call the communicator is aborted (peers fail instead of
 * hanging) and further sharded calls on this context return NACS_ENCCL. */
nacs_status nacs_create_sharded(nacs_ctx **out, int device, void *cuda_stream, const void *nccl_unique_id,
                                int rank, int world);
/* Write a fresh ncclUniqueId (128 bytes) to out. */
nacs_status nacs_nccl_unique_id(void *out);
void nacs_destroy(nacs_ctx *ctx);

/* Load (or replace) the DC state.  Validates k, capacities and residual ranges. */
nacs_status nacs_load_topology(nacs_ctx *ctx, const nacs_topology *topo);

/* Copy the current state back to host arrays (any may be NULL): cpu_res[n], ram_res[n],
 * active[n], link_res[L]. */
nacs_status nacs_read_topology(nacs_ctx *ctx, int32_t *cpu_res, int32_t *ram_res, uint8_t *active,
                               int32_t *link_res);

/* Rank every server for one pod step on the current state (no state change):
 * feasibility filter (Eq. 4-7, R6) then AHP (Eq. 9-10, R7-R11) or
 * TOPSIS (R12-R13) scores over the feasible set, then the argmax with the
 * lowest server index on ties (R14).  mask[n] (uint8, may be NULL): 1 = feasible.
 * scores[n] (float, may be NULL): the FP32 score of feasible servers, 0 elsewhere.
 * best: the chosen server, -1 if none is feasible.  Device pointers (NACS_DEVICE_PTRS):
 * scores 16-byte aligned, mask 4-byte aligned (else NACS_EINVAL). */
nacs_status nacs_rank_ahp(nacs_ctx *ctx, const nacs_options *opt, const nacs_pod_query *q, uint8_t *mask,
                          float *scores, int32_t *best);
nacs_status nacs_rank_topsis(nacs_ctx *ctx, const nacs_options *opt, const nacs_pod_query *q,
                             uint8_t *mask, float *scores, int32_t *best);

/* Whole-GPU TOPSIS ranking of ONE pod step on each of n_states DC states (SURVEY 8(d):
 * "standalone nacs_rank_topsis on cold snapshots"; the same filter, statistics, closeness
 * and argmax as nacs_rank_topsis: Eq. 4-7, R4-R6, R12-R14).  Every
 * state is ranked independently for the same query q (pod demand, flows, exclusions).
 * states: n_states DC states of the loaded topology's geometry and capacities, each the
 * int32 words cpu_res[n] | ram_res[n] | active[n] (0/1) | link_res[L] (canonical link order),
 * consecutive states state_stride >= 3n + L words apart; the loaded state is not used.
 * Outputs: mask [n_states][n] (uint8, may be NULL), scores [n_states][n] (FP32 closeness of
 * feasible servers, 0 elsewhere; may be NULL), best [n_states] (argmax, lowest index on ties;
 * -1 if no server is feasible; -2 if the state holds a residual outside [0, capacity] or an
 * f_u outside {0, 1}, in which case the call returns NACS_EINVAL unless NACS_ASYNC).
 * NACS_DEVICE_PTRS: states and outputs are device pointers (the streaming form: one launch,
 * a thread-block cluster per state) — states and scores 16-byte aligned, mask and best 4-byte
 * aligned, state_stride even (a multiple of 4 takes the TMA path) — else NACS_EINVAL;
 * otherwise host arrays, staged through device buffers.
 * Flow/exclusion arrays of q follow the same flag.  TOPSIS only, bw_criterion = NACS_BW_ACCESS,
 * n <= 65536, not on server-sharded contexts.  Stats: pod_steps = n_states. */
nacs_status nacs_rank_topsis_many(nacs_ctx *ctx, const nacs_options *opt, const nacs_pod_query *q, int32_t n_states,
                                  const int32_t *states, int64_t state_stride, uint8_t *mask, float *scores,
                                  int32_t *best);

/* Schedule requests one after another against the live state (the paper's online
 * semantics): for each pod in ascending id, rank, select, and commit
 * (Eq. 4-5, R16-R18); at request end top up allocations (R19).  An accepted request
 * stays committed; a rejected one leaves the state unchanged (R20). */
nacs_status nacs_schedule_request(nacs_ctx *ctx, const nacs_options *opt, const nacs_requests *reqs,
                                  nacs_placements *out);

/* Schedule every request of the batch against the same current state, each with its own
 * private overlay (R21): requests do not see each other and the state is not modified. */
nacs_status nacs_schedule_batch(nacs_ctx *ctx, const nacs_options *opt, const nacs_requests *batch,
                                nacs_placements *out);

/* ---------------------------------------------------------------------------------------
 * Departures and the discrete-event simulator: "a discrete event
 * simulator" drives the scheduler; the E2 campaign and its
 * metrics "# Events", runtime, U(ij), U(i) (T5 P:416-426), fragmentation F(N^s), F(E^s)
 * (P:111-112).
 * ------------------------------------------------------------------------------------- */

/* Release the accepted requests (status 1) of a batch the context scheduled earlier
 * (nacs_schedule_request): every container's c^a and every vlink's bw^a return to the
 * state (the exact inverse of commit and top-up); f_u of the touched servers is re-derived
 * as "some residual below capacity" (R22).  reqs/pl: the batch and its placements as
 * returned.  flags: NACS_DEVICE_PTRS | NACS_ASYNC.  A placement that does not match the
 * fat-tree, or a release that would raise a residual above its capacity (e.g. released
 * twice), fails with NACS_EINVAL and changes nothing (without NACS_ASYNC). */
nacs_status nacs_release(nacs_ctx *ctx, uint32_t flags, const nacs_requests *reqs, const nacs_placements *pl);

typedef struct {
  int32_t max_ticks;     /* the run ends after this many ticks at the latest (>= 1) */
  int32_t hol_blocking;  /* 1: FIFO with head-of-line blocking; 0: scan the whole queue */
} nacs_sim_config;

typedef struct {  /* caller-allocated arrays; scalars written by the call */
  int32_t *start_tick;    /* [n_requests] tick of acceptance, -1 if never accepted */
  int32_t *attempts;      /* [n_requests] scheduling attempts */
  int32_t *tick_servers;  /* [max_ticks] active servers |N^s'| after each tick */
  int32_t *tick_links;    /* [max_ticks] active links |E^s'| (residual below capacity) */
  int32_t *tick_queue;    /* [max_ticks] queued requests after each tick */
  int64_t events;         /* ticks simulated (T5 "# Events"; entries >= events untouched) */
  int64_t attempts_total; /* scheduler invocations */
  int64_t accepted;
  double sched_seconds;   /* device time of the event loop (one kernel: every attempt and departure; T5 "runtime") */
  double wall_seconds;    /* wall time of the whole call */
} nacs_sim_report;

/* Discrete-event simulation on the context's live state (reading R28).  Ticks t = 0, 1, ...:
 * (1) the requests whose start + duration == t depart (nacs_release); (2) the requests with
 * arrival == t join the queue in ascending id; (3) queued requests are offered in FIFO order
 * to the scheduler (nacs_schedule_request semantics with opt); an accepted request leaves
 * the queue and holds its resources for duration ticks; a refused one stays queued (with
 * hol_blocking the scan of the tick stops there).  The run ends after the first tick with
 * an empty queue and no arrival left, or after max_ticks (still-queued requests are then
 * rejected).  out: the final placements (status 1 accepted, 0 never accepted, -1 invalid).
 * Afterwards the state holds the requests that have not departed.  The whole event loop
 * runs on the device in one launch (one CTA: queue, running set and every attempt on-chip).
 * Host pointers only; synchronous; arrival >= 0, duration >= 1; AHP/TOPSIS/BF/WF with
 * rank_mode per pod. */
nacs_status nacs_simulate(nacs_ctx *ctx, const nacs_options *opt, const nacs_requests *reqs, const int32_t *arrival,
                          const int32_t *duration, const nacs_sim_config *cfg, nacs_placements *out,
                          nacs_sim_report *rep);

/* ---------------------------------------------------------------------------------------
 * General topology.  "A modified Dijkstra algorithm is used to compute
 * the shortest path that has the maximum available bandwidth between the hosting servers
 * ... each thread calculates a different source and destination pair" (§V-D),
 * for a DC G^s(N^s, E^s) given as an arbitrary undirected graph (§II-A) instead of
 * a fat-tree.  Reading R26: a link is usable by a flow of demand D iff its residual >= D;
 * the returned path has the fewest hops over usable links, then the largest bottleneck
 * (minimum residual along it), then the lexicographically smallest vertex sequence.
 * ------------------------------------------------------------------------------------- */
#define NACS_MAX_GRAPH_VERTICES 16777216  /* 2^24 */
#define NACS_MAX_GRAPH_LINKS 268435456    /* 2^28 */

/* Vertices 0..n_vertices-1, of which 0..n_servers-1 are the servers; link l joins link_u[l]
 * and link_v[l] (undirected; parallel links allowed, no self-loops) with residual
 * bandwidth link_res[l] in [0, NACS_MAX_CAP] Mbps.  Host pointers.  Independent of the
 * fat-tree state of nacs_load_topology; a context holds one of each. */
typedef struct {
  int32_t n_vertices;   /* 2..NACS_MAX_GRAPH_VERTICES */
  int32_t n_servers;    /* 1..n_vertices */
  int32_t n_links;      /* 0..NACS_MAX_GRAPH_LINKS */
  const int32_t *link_u, *link_v, *link_res;
} nacs_graph;

/* Queries: path i goes from src[i] to dst[i] (vertex ids, src != dst) for a flow of
 * demand[i] in [0, NACS_MAX_CAP] Mbps. */
typedef struct {
  int32_t n_queries;
  const int32_t *src, *dst, *demand;
} nacs_path_query;

/* Load (or replace) the graph.  Validates endpoints, self-loops and residual ranges. */
nacs_status nacs_load_graph(nacs_ctx *ctx, const nacs_graph *g);

/* Widest-shortest path of every query on the loaded graph, all against the same graph
 * (queries are independent).  Outputs (caller-allocated, [n_queries]):
 * bottleneck[i] = minimum residual along the path, hops[i] = its link count; both -1 when
 * no usable path exists.  path (may be NULL): [n_queries][max_hops + 1] vertex ids
 * src..dst, -1 padded; a row is all -1 if the query is infeasible or hops[i] > max_hops.
 * flags: NACS_DEVICE_PTRS (all five arrays on the device; invalid queries then get
 * hops = -2 and the call returns NACS_EINVAL after the kernel unless NACS_ASYNC) |
 * NACS_ASYNC.  Host pointers: invalid queries (endpoint out of range, src == dst, demand
 * out of range) fail the call with NACS_EINVAL before any work. */
nacs_status nacs_widest_paths(nacs_ctx *ctx, const nacs_path_query *q, uint32_t flags, int32_t *bottleneck,
                              int32_t *hops, int32_t *path, int32_t max_hops);

/* Logical bandwidth criterion (reading R2's alternative: "sum of all bandwidth capacity
 * bw^s_uv with source on u"): out[u] (int64, [n_servers]) = sum over the servers
 * v != u of the bottleneck of the widest shortest u-v path with every link usable;
 * unreachable servers add 0.  flags: NACS_DEVICE_PTRS | NACS_ASYNC. */
nacs_status nacs_logical_bandwidth(nacs_ctx *ctx, uint32_t flags, int64_t *out);

nacs_status nacs_last_stats(nacs_ctx *ctx, nacs_stats *out);
const char *nacs_last_error(const nacs_ctx *ctx);

#ifdef __cplusplus
}
#endif

#endif /* NACS_H */
