// nacs_api.cu — the C ABI of libnacs (include/nacs.h): context, validation, staging of
// inputs and outputs, kernel launches.  Every step of the method runs in the kernels of
// nacs_kernels.cu; this file only checks arguments and moves bytes.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <chrono>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include <nccl.h>
#include <nvtx3/nvToolsExt.h>  // header-only: ranges are free unless a profiler is attached

#include "../../include/nacs.h"
#include "nacs_internal.h"

using nacs::Geo;
using nacs::Opt;

namespace {

template <class T>
struct DevArr {
  T* p = nullptr;
  size_t cap = 0;
  cudaError_t reserve(size_t n) {
    if (n <= cap) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    size_t m = n + n / 4 + 64;
    cudaError_t e = cudaMalloc(&p, m * sizeof(T));
    if (e == cudaSuccess) cap = m;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

struct PinArr {  // page-locked, mapped: dp is the device view (zero-copy outputs)
  unsigned char* p = nullptr;
  unsigned char* dp = nullptr;
  size_t cap = 0;
  cudaError_t reserve(size_t n) {
    if (n <= cap) return cudaSuccess;
    if (p) cudaFreeHost(p);
    p = dp = nullptr;
    cap = 0;
    size_t m = n + n / 4 + 4096;
    cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&p), m, cudaHostAllocMapped);
    if (e == cudaSuccess) e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&dp), p, 0);
    if (e == cudaSuccess) cap = m;
    return e;
  }
  void release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
  }
};

}  // namespace

struct nacs_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  bool has_topo = false;
  Geo g{};
  int num_sms = 0;
  DevArr<int> state;
  DevArr<int> req_in;        // packed CSR inputs
  DevArr<int> req_out;       // packed outputs
  DevArr<int2> ulog;
  DevArr<int4> wlog;         // per-warp undo logs of k_batch_warp
  DevArr<int> wlay;          // chunk layout of the snapshot for k_batch_warp
  DevArr<int> deferred;      // requests k_batch_warp hands to k_batch
  DevArr<double> w64;
  DevArr<float> ahp_ws;
  DevArr<unsigned char> ahp_glob;  // AHP batch workspace in global memory (k_batch, large n)
  DevArr<unsigned long long> seqc; // k_seq_cluster exchange: statistics, keys, FP64 candidates
  DevArr<int> misc;          // next-request counter, query arrays, best
  DevArr<unsigned char> mask;
  DevArr<float> scores;
  DevArr<unsigned long long> stats;
  PinArr pin_in, pin_out;
  std::string err;
  nacs_stats last{};
  bool stats_pending = false;
  bool cta_only = false;     // NACS_CTA_ONLY=1: force the CTA-per-request batch kernel (testing)
  // server sharding (nacs_create_sharded)
  int rank = 0, world = 1;
  bool loopback = false;
  bool comm_aborted = false;  // an error inside a sharded call aborted the communicator
  ncclComm_t comm = nullptr;
  DevArr<unsigned char> sh_buf;
  PinArr sh_ctl;
  // general topology (nacs_load_graph): CSR adjacency, path-kernel scratch and staging
  bool has_graph = false;
  int gV = 0, gns = 0, gL = 0;
  DevArr<int> g_off;
  DevArr<int2> g_adj;
  DevArr<unsigned> g_adj16;
  bool g_packed = false;
  DevArr<unsigned> g_scratch;
  DevArr<int> g_io;
  DevArr<long long> g_out;
  DevArr<int> g_ws;
  DevArr<int> crit;          // logical-bandwidth criteria table (nacs_rank_*, bw_criterion = 1)
  DevArr<int> many;          // nacs_rank_topsis_many host-pointer staging: states | best
  DevArr<unsigned char> many_mask;
  DevArr<float> many_scores;
  // departures / simulator
  DevArr<long long> rel_delta;
  DevArr<int> sim_buf;
  PinArr sim_pin;
};

namespace {

// NVTX range over one API call (tracing): nsys / ncu --nvtx see every call
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

nacs_status fail(nacs_ctx* c, nacs_status s, const std::string& msg) {
  if (c) c->err = msg;
  return s;
}

nacs_status cuda_fail(nacs_ctx* c, cudaError_t e, const char* where) {
  std::string m = std::string(where) + ": " + cudaGetErrorString(e);
  cudaGetLastError();
  return fail(c, e == cudaErrorMemoryAllocation ? NACS_ENOMEM : NACS_ECUDA, m);
}

#define CK(call)                                              \
  do {                                                        \
    cudaError_t e_ = (call);                                  \
    if (e_ != cudaSuccess) return cuda_fail(ctx, e_, #call);  \
  } while (0)

nacs_status check_options(nacs_ctx* ctx, const nacs_options* o, Opt* out) {
  if (!o) return fail(ctx, NACS_EINVAL, "options: NULL");
  std::string m;
  if (o->method < NACS_AHP || o->method > NACS_WF) m += "options.method not AHP/TOPSIS/BF/WF; ";
  double sum = 0;
  for (int k = 0; k < 4; ++k) {
    if (!std::isfinite(o->weights[k]) || o->weights[k] < 0) m += "options.weights[" + std::to_string(k) + "] not finite and >= 0; ";
    sum += o->weights[k];
  }
  if (!(std::fabs(sum - 1.0) <= 1e-6)) m += "options.weights do not sum to 1 (|sum-1| > 1e-6); ";
  if (o->ahp_rule != 0 && o->ahp_rule != 1) m += "options.ahp_rule not 0/1; ";
  if (o->l1_mode != 0 && o->l1_mode != 1) m += "options.l1_mode not 0/1; ";
  if (o->path_filter != 0 && o->path_filter != 1) m += "options.path_filter not 0/1; ";
  if (o->flags & ~(NACS_DEVICE_PTRS | NACS_ASYNC | NACS_EXACT_FP64)) m += "options.flags has unknown bits; ";
  if (o->rank_mode != NACS_RANK_PER_POD && o->rank_mode != NACS_RANK_ONCE) m += "options.rank_mode not 0/1; ";
  if (o->method >= NACS_BF && o->rank_mode == NACS_RANK_ONCE) m += "options.rank_mode = NACS_RANK_ONCE needs AHP/TOPSIS; ";
  if (o->bw_criterion != NACS_BW_ACCESS && o->bw_criterion != NACS_BW_LOGICAL) m += "options.bw_criterion not 0/1; ";
  if (!m.empty()) return fail(ctx, NACS_EINVAL, m);
  out->method = (int)o->method;
  for (int k = 0; k < 4; ++k) out->wd[k] = o->weights[k];
  out->ahp_rule = o->ahp_rule;
  out->l1_mode = o->l1_mode;
  // BF / WF ignore the network at selection and route afterwards (R27)
  out->path_filter = o->method >= NACS_BF ? 0 : o->path_filter;
  out->exact64 = (o->flags & NACS_EXACT_FP64) ? 1 : 0;
  out->rank_once = o->rank_mode == NACS_RANK_ONCE;
  out->bw_logical = o->bw_criterion == NACS_BW_LOGICAL;
  return NACS_OK;
}

// Host-side validation of a host-pointer CSR batch (R24).  Lists every violation.
// Host-side work of the host-pointer path (validation, staging copies) split over up to 16
// threads: at C4 a batch is 42 MB in and 24 MB out, which one core copies at ~10 GB/s.
static int host_threads(size_t work, size_t grain) {
  const unsigned hw = std::thread::hardware_concurrency();
  size_t t = work / grain;
  if (t > 16) t = 16;
  if (t > hw && hw > 0) t = hw;
  return t < 1 ? 1 : (int)t;
}
// A process-wide pool of 15 host workers (created on first use; dispatches serialised).
class HostPool {
 public:
  static HostPool& get() {
    static HostPool* pool = new HostPool(15);  // never destroyed: workers live with the process
    return *pool;
  }
  // job(t) for t in [0, nt), nt <= 16; the caller runs t = 0
  void run(int nt, const std::function<void(int)>& job) {
    std::lock_guard<std::mutex> call(call_mu_);
    {
      std::lock_guard<std::mutex> lk(mu_);
      job_ = &job;
      want_ = nt - 1;
      done_ = 0;
      ++gen_;
    }
    cv_.notify_all();
    job(0);
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return done_ == want_; });
    job_ = nullptr;
  }

 private:
  explicit HostPool(int n) {
    for (int i = 0; i < n; ++i) std::thread([this, i] { loop(i + 1); }).detach();
  }
  void loop(int id) {
    unsigned long long seen = 0;
    for (;;) {
      const std::function<void(int)>* job;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        if (id > want_) continue;
        job = job_;
      }
      (*job)(id);
      {
        std::lock_guard<std::mutex> lk(mu_);
        ++done_;
      }
      done_cv_.notify_one();
    }
  }
  std::mutex call_mu_, mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)>* job_ = nullptr;
  int want_ = 0, done_ = 0;
  unsigned long long gen_ = 0;
};

template <typename F>
static void parallel_ranges(size_t n, int nt, F fn) {  // fn(thread, begin, end), contiguous ranges
  if (nt <= 1) { fn(0, (size_t)0, n); return; }
  HostPool::get().run(nt, [&](int t) { fn(t, n * t / nt, n * (t + 1) / nt); });
}
struct CopyJob {
  void* dst;
  const void* src;
  size_t bytes;
};
// The jobs as one concatenated byte range split evenly over the threads.
static void parallel_copies(const std::vector<CopyJob>& jobs) {
  size_t total = 0;
  for (auto& j : jobs) total += j.bytes;
  parallel_ranges(total, host_threads(total, (size_t)1 << 21), [&](int, size_t b, size_t e) {
    size_t at = 0;
    for (auto& j : jobs) {
      const size_t lo = std::max(b, at), hi = std::min(e, at + j.bytes);
      if (lo < hi) std::memcpy(static_cast<char*>(j.dst) + (lo - at), static_cast<const char*>(j.src) + (lo - at), hi - lo);
      at += j.bytes;
    }
  });
}

// Structure of a host CSR batch (NULL arrays, offsets): what sizing the copies needs.
nacs_status check_offsets_host(nacs_ctx* ctx, const nacs_requests* q, int* C_out, int* V_out) {
  if (!q) return fail(ctx, NACS_EINVAL, "requests: NULL");
  if (q->n_requests < 0) return fail(ctx, NACS_EINVAL, "requests.n_requests < 0");
  int R = q->n_requests;
  if (R == 0) { *C_out = *V_out = 0; return NACS_OK; }
  if (!q->container_off || !q->vlink_off || !q->cpu_min || !q->cpu_max || !q->ram_min || !q->ram_max ||
      !q->pod_of)
    return fail(ctx, NACS_EINVAL, "requests: NULL array");
  if (q->container_off[0] != 0 || q->vlink_off[0] != 0)
    return fail(ctx, NACS_EINVAL, "requests: offsets must start at 0");
  for (int r = 0; r < R; ++r) {  // offsets first (they size every array)
    if (q->container_off[r + 1] < q->container_off[r] || q->vlink_off[r + 1] < q->vlink_off[r])
      return fail(ctx, NACS_EINVAL, "request " + std::to_string(r) + ": decreasing offsets");
  }
  if (q->vlink_off[R] > 0 && (!q->vl_src || !q->vl_dst || !q->bw_min || !q->bw_max))
    return fail(ctx, NACS_EINVAL, "requests: NULL vlink array");
  *C_out = q->container_off[R];
  *V_out = q->vlink_off[R];
  return NACS_OK;
}

// Every request of a host batch (R24, sizes), in parallel; the messages name the first
// invalid requests in request order.  Call after check_offsets_host.
nacs_status validate_requests_host(nacs_ctx* ctx, const nacs_requests* q) {
  const int R = q->n_requests;
  const int nt = host_threads((size_t)R, 4096);
  struct Part {
    int nbad = 0;
    bool big = false;
    std::string m;
  };
  std::vector<Part> parts(nt);
  parallel_ranges((size_t)R, nt, [&](int t, size_t rb, size_t re) {
    Part& P = parts[t];
    for (int r = (int)rb; r < (int)re; ++r) {
      const int c0 = q->container_off[r], c1 = q->container_off[r + 1];
      const int v0 = q->vlink_off[r], v1 = q->vlink_off[r + 1];
      const int bad = nacs::validate_request(c1 - c0, v1 - v0, q->cpu_min + c0, q->cpu_max + c0, q->ram_min + c0,
                                             q->ram_max + c0, q->pod_of + c0, q->vl_src + v0, q->vl_dst + v0,
                                             q->bw_min + v0, q->bw_max + v0);
      if (!bad) continue;
      ++P.nbad;
      if (bad & 1) P.big = true;
      if (P.nbad <= 32) {
        P.m += "request " + std::to_string(r) + ":";
        if (bad & 1) P.m += " size (containers 1.." + std::to_string(nacs::MAXC) + ", vlinks <= " +
                            std::to_string(nacs::MAXV) + ")";
        if (bad & 2) P.m += " non-positive c^min";
        if (bad & 4) P.m += " c^min > c^max";
        if (bad & 8) P.m += " pod ids not 0..P-1";
        if (bad & 16) P.m += " vlink endpoint out of range or self-loop";
        if (bad & 32) P.m += " bw^min <= 0 or bw^min > bw^max";
        P.m += "; ";
      }
    }
  });
  std::string m;
  int nbad = 0;
  bool big = false;
  for (auto& P : parts) {  // messages of the first invalid requests, in request order
    if (nbad < 32) m += P.m;
    nbad += P.nbad;
    big |= P.big;
  }
  if (nbad) {
    if (nbad > 32) m += "... " + std::to_string(nbad) + " invalid requests in total";
    return fail(ctx, big ? NACS_ETOOBIG : NACS_EINVAL, m);
  }
  return NACS_OK;
}

nacs_status check_requests_host(nacs_ctx* ctx, const nacs_requests* q, int* C_out, int* V_out) {
  nacs_status st = check_offsets_host(ctx, q, C_out, V_out);
  if (st || q->n_requests == 0) return st;
  return validate_requests_host(ctx, q);
}

nacs_status check_placements(nacs_ctx* ctx, const nacs_placements* o) {
  if (!o || !o->status || !o->server_of_container || !o->cpu_alloc || !o->ram_alloc || !o->bw_alloc ||
      !o->path_of_vlink)
    return fail(ctx, NACS_EINVAL, "placements: NULL array");
  return NACS_OK;
}

// Stage a host CSR batch into device memory with one copy; returns device views.
nacs_status stage_requests(nacs_ctx* ctx, const nacs_requests* q, int C, int V, nacs::ReqsDev* R) {
  int Rn = q->n_requests;
  size_t words = 2 * (size_t)(Rn + 1) + 5 * (size_t)C + 4 * (size_t)V;
  CK(ctx->pin_in.reserve(words * 4));
  CK(ctx->req_in.reserve(words));
  int* h = reinterpret_cast<int*>(ctx->pin_in.p);
  size_t o = 0;
  std::vector<CopyJob> jobs;
  auto put = [&](const int32_t* src, size_t n) {
    size_t at = o;
    if (n) jobs.push_back({h + o, src, n * 4});
    o += n;
    return at;
  };
  size_t a_coff = put(q->container_off, Rn + 1), a_voff = put(q->vlink_off, Rn + 1);
  size_t a_cmin = put(q->cpu_min, C), a_cmax = put(q->cpu_max, C), a_rmin = put(q->ram_min, C);
  size_t a_rmax = put(q->ram_max, C), a_pod = put(q->pod_of, C);
  size_t a_src = put(q->vl_src, V), a_dst = put(q->vl_dst, V), a_bmin = put(q->bw_min, V), a_bmax = put(q->bw_max, V);
  // in 4 pieces: the copy engine moves piece i while the host threads fill piece i + 1
  const size_t total = words * 4, piece = ((total / 4) + 4095) & ~(size_t)4095;
  for (size_t b = 0; b < total; b += piece) {
    const size_t e = std::min(total, b + piece);
    std::vector<CopyJob> part;
    size_t at = 0;
    for (auto& j : jobs) {
      const size_t lo = std::max(b, at), hi = std::min(e, at + j.bytes);
      if (lo < hi)
        part.push_back({static_cast<char*>(j.dst) + (lo - at), static_cast<const char*>(j.src) + (lo - at), hi - lo});
      at += j.bytes;
    }
    parallel_copies(part);
    CK(cudaMemcpyAsync(reinterpret_cast<char*>(ctx->req_in.p) + b, reinterpret_cast<const char*>(h) + b, e - b,
                       cudaMemcpyHostToDevice, ctx->stream));
  }
  int* d = ctx->req_in.p;
  R->n = Rn;
  R->coff = d + a_coff;
  R->voff = d + a_voff;
  R->cpu_min = d + a_cmin;
  R->cpu_max = d + a_cmax;
  R->ram_min = d + a_rmin;
  R->ram_max = d + a_rmax;
  R->pod_of = d + a_pod;
  R->src = d + a_src;
  R->dst = d + a_dst;
  R->bw_min = d + a_bmin;
  R->bw_max = d + a_bmax;
  return NACS_OK;
}

nacs::ReqsDev device_requests(const nacs_requests* q) {
  nacs::ReqsDev R;
  R.n = q->n_requests;
  R.coff = q->container_off;
  R.voff = q->vlink_off;
  R.cpu_min = q->cpu_min;
  R.cpu_max = q->cpu_max;
  R.ram_min = q->ram_min;
  R.ram_max = q->ram_max;
  R.pod_of = q->pod_of;
  R.src = q->vl_src;
  R.dst = q->vl_dst;
  R.bw_min = q->bw_min;
  R.bw_max = q->bw_max;
  return R;
}

nacs_status device_outputs(nacs_ctx* ctx, int R, int C, int V, nacs::OutDev* O) {
  size_t words = (size_t)R + 3 * (size_t)C + 2 * (size_t)V;
  CK(ctx->req_out.reserve(words + 1));
  int* d = ctx->req_out.p;
  O->status = d;
  O->server = d + R;
  O->cpu_a = d + R + C;
  O->ram_a = d + R + 2 * (size_t)C;
  O->bw_a = d + R + 3 * (size_t)C;
  O->path = d + R + 3 * (size_t)C + V;
  return NACS_OK;
}

// Outputs straight into mapped page-locked memory (the kernels write them over the bus as
// requests finish; no device-to-host copy after the kernels).
nacs_status mapped_outputs(nacs_ctx* ctx, int R, int C, int V, nacs::OutDev* O) {
  size_t words = (size_t)R + 3 * (size_t)C + 2 * (size_t)V;
  CK(ctx->pin_out.reserve(words * 4 + 4));
  int* d = reinterpret_cast<int*>(ctx->pin_out.dp);
  O->status = d;
  O->server = d + R;
  O->cpu_a = d + R + C;
  O->ram_a = d + R + 2 * (size_t)C;
  O->bw_a = d + R + 3 * (size_t)C;
  O->path = d + R + 3 * (size_t)C + V;
  return NACS_OK;
}
void copy_mapped_outputs(nacs_ctx* ctx, int R, int C, int V, nacs_placements* out) {
  const int* h = reinterpret_cast<const int*>(ctx->pin_out.p);
  parallel_copies({{out->status, h, (size_t)R * 4},
                   {out->server_of_container, h + R, (size_t)C * 4},
                   {out->cpu_alloc, h + R + C, (size_t)C * 4},
                   {out->ram_alloc, h + R + 2 * (size_t)C, (size_t)C * 4},
                   {out->bw_alloc, h + R + 3 * (size_t)C, (size_t)V * 4},
                   {out->path_of_vlink, h + R + 3 * (size_t)C + V, (size_t)V * 4}});
}

nacs_status unstage_outputs(nacs_ctx* ctx, int R, int C, int V, nacs_placements* out) {
  size_t words = (size_t)R + 3 * (size_t)C + 2 * (size_t)V;
  CK(ctx->pin_out.reserve(words * 4 + 4));
  CK(cudaMemcpyAsync(ctx->pin_out.p, ctx->req_out.p, words * 4, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  const int* h = reinterpret_cast<const int*>(ctx->pin_out.p);
  parallel_copies({{out->status, h, (size_t)R * 4},
                   {out->server_of_container, h + R, (size_t)C * 4},
                   {out->cpu_alloc, h + R + C, (size_t)C * 4},
                   {out->ram_alloc, h + R + 2 * (size_t)C, (size_t)C * 4},
                   {out->bw_alloc, h + R + 3 * (size_t)C, (size_t)V * 4},
                   {out->path_of_vlink, h + R + 3 * (size_t)C + V, (size_t)V * 4}});
  return NACS_OK;
}

nacs_status begin_call(nacs_ctx* ctx) {
  if (!ctx) return NACS_EINVAL;
  ctx->err.clear();
  CK(cudaSetDevice(ctx->device));
  if (!ctx->has_topo) return fail(ctx, NACS_ENOTOPO, "no topology loaded");
  CK(ctx->stats.reserve(nacs::ST_N));
  CK(cudaMemsetAsync(ctx->stats.p, 0, sizeof(unsigned long long) * nacs::ST_N, ctx->stream));
  ctx->stats_pending = true;
  return NACS_OK;
}

nacs_status finish_stats(nacs_ctx* ctx) {
  if (!ctx->stats_pending) return NACS_OK;
  unsigned long long h[nacs::ST_N];
  CK(cudaMemcpyAsync(h, ctx->stats.p, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->last.pod_steps = (int64_t)h[nacs::ST_POD_STEPS];
  ctx->last.servers_ranked = (int64_t)h[nacs::ST_POD_STEPS] * ctx->g.n;
  ctx->last.retries = (int64_t)h[nacs::ST_RETRIES];
  ctx->last.fp64_decisions = (int64_t)h[nacs::ST_FP64];
  ctx->last.invalid = (int64_t)h[nacs::ST_INVALID];
  ctx->last.feasible = (int64_t)h[nacs::ST_FEAS];
  ctx->last.ahp_pairs = (int64_t)h[nacs::ST_PAIRS];
  ctx->last.scanned_a = (int64_t)h[nacs::ST_SCAN_A];
  ctx->last.scanned_b = (int64_t)h[nacs::ST_SCAN_B];
  ctx->last.edges_scanned = (int64_t)h[nacs::ST_EDGES];
  ctx->last.bfs_runs = (int64_t)h[nacs::ST_BFS];
  ctx->stats_pending = false;
  return NACS_OK;
}

nacs::RankManyArgs rank_many_args(nacs_ctx* ctx, const Opt& o, const nacs::QueryDev& qd, const int* states,
                                   long long stride, int B) {
  nacs::RankManyArgs a{};
  a.g = ctx->g;
  for (int c = 0; c < 4; ++c) a.wd[c] = o.wd[c];
  a.path_filter = o.path_filter;
  a.exact64 = o.exact64;
  a.states = states;
  a.stride = stride;
  a.B = B;
  a.dc = qd.dc;
  a.dr = qd.dr;
  a.nflow = qd.nflow;
  a.nex = qd.nex;
  a.fv = qd.fv;
  a.fD = qd.fD;
  a.ex = qd.ex;
  a.mask = qd.mask;
  a.scores = qd.scores;
  a.best = qd.best;
  a.stats = ctx->stats.p;
  return a;
}

// Host-side checks of a pod query (nacs_rank_*); copies host flows (sorted by server) and
// exclusions to the device, or takes device pointers as given.
nacs_status query_device(nacs_ctx* ctx, const nacs_pod_query* q, bool dev, nacs::QueryDev* qd) {
  const Geo& g = ctx->g;
  std::string m;
  if (q->cpu_demand <= 0 || q->ram_demand <= 0) m += "query demands must be > 0; ";
  if (q->n_flows < 0 || q->n_flows > nacs::MAXF) m += "query.n_flows out of 0..128; ";
  if (q->n_excluded < 0 || q->n_excluded > g.n) m += "query.n_excluded out of range; ";
  if (q->n_flows > 0 && (!q->flow_server || !q->flow_bw)) m += "query flow arrays NULL; ";
  if (q->n_excluded > 0 && !q->excluded) m += "query.excluded NULL; ";
  if (!m.empty()) return fail(ctx, NACS_EINVAL, m);
  int nf = q->n_flows, nx = q->n_excluded;
  CK(ctx->misc.reserve(2 * (size_t)nf + nx + 8));
  qd->dc = q->cpu_demand;
  qd->dr = q->ram_demand;
  qd->nflow = nf;
  qd->nex = nx;
  qd->crit = nullptr;
  if (dev) {
    qd->fv = q->flow_server;
    qd->fD = q->flow_bw;
    qd->ex = q->excluded;
    return NACS_OK;
  }
  std::vector<int> fv(q->flow_server, q->flow_server + nf), fD(q->flow_bw, q->flow_bw + nf);
  for (int f = 0; f < nf; ++f) {
    if (fv[f] < 0 || fv[f] >= g.n) m += "flow " + std::to_string(f) + ": server out of range; ";
    if (fD[f] <= 0) m += "flow " + std::to_string(f) + ": demand <= 0; ";
  }
  std::vector<int> idx(nf);
  for (int f = 0; f < nf; ++f) idx[f] = f;
  std::sort(idx.begin(), idx.end(), [&](int a, int b) { return fv[a] < fv[b]; });
  std::vector<int> h(2 * (size_t)nf + nx + 1);
  for (int f = 0; f < nf; ++f) {
    h[f] = fv[idx[f]];
    h[nf + f] = fD[idx[f]];
    if (f && h[f] == h[f - 1]) m += "flow servers not distinct; ";
  }
  for (int i = 0; i < nx; ++i) {
    h[2 * nf + i] = q->excluded[i];
    if (q->excluded[i] < 0 || q->excluded[i] >= g.n) m += "excluded server out of range; ";
  }
  if (!m.empty()) return fail(ctx, NACS_EINVAL, m);
  CK(cudaMemcpyAsync(ctx->misc.p + 4, h.data(), h.size() * 4, cudaMemcpyHostToDevice, ctx->stream));
  qd->fv = ctx->misc.p + 4;
  qd->fD = ctx->misc.p + 4 + nf;
  qd->ex = ctx->misc.p + 4 + 2 * nf;
  return NACS_OK;
}

nacs_status rank_impl(nacs_ctx* ctx, const nacs_options* opt, const nacs_pod_query* q, uint8_t* mask,
                      float* scores, int32_t* best, int method) {
  nacs_status st = begin_call(ctx);
  if (st) return st;
  Opt o;
  if ((st = check_options(ctx, opt, &o))) return st;
  if (o.method != method) return fail(ctx, NACS_EINVAL, "options.method does not match the rank call");
  if (!q || !best) return fail(ctx, NACS_EINVAL, "query/best: NULL");
  const bool dev = opt->flags & NACS_DEVICE_PTRS;
  const Geo& g = ctx->g;
  nacs::QueryDev qd{};
  if ((st = query_device(ctx, q, dev, &qd))) return st;
  CK(ctx->mask.reserve(g.n));
  CK(ctx->scores.reserve(g.n));
  if (dev && (((uintptr_t)scores % 16) || ((uintptr_t)mask % 4)))
    return fail(ctx, NACS_EINVAL, "device scores must be 16-byte aligned and mask 4-byte aligned");
  qd.mask = (dev && mask) ? mask : ctx->mask.p;
  qd.scores = (dev && scores) ? scores : ctx->scores.p;
  qd.best = dev ? best : ctx->misc.p;
  qd.crit = nullptr;
  if (o.bw_logical) {  // R2's logical reading of the Bandwidth criterion
    if (ctx->world > 1 || ctx->comm)
      return fail(ctx, NACS_EINVAL, "options.bw_criterion = NACS_BW_LOGICAL is not available on server-sharded contexts");
    CK(ctx->crit.reserve(4 * (size_t)g.n + (size_t)g.E * g.E + 4));
    int* crit = ctx->crit.p;
    int* F = crit + 4 * (size_t)g.n;
    int* tb = F + (size_t)g.E * g.E;
    CK(nacs::launch_logical_criteria(g, ctx->state.p, crit, F, tb, ctx->stream));
    int too_big = 0;
    CK(cudaMemcpyAsync(&too_big, tb, 4, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (too_big)
      return fail(ctx, NACS_ETOOBIG, "logical bandwidth >= 2^24 (n x link_cap too large to be exact in FP32, R5)");
    qd.crit = crit;
  }
  if (method == 0) {
    CK(ctx->ahp_ws.reserve(nacs::ahp_workspace_bytes(g.n) / 4 + 4));
    CK(ctx->w64.reserve(nacs::ahp_workspace_doubles(g.n)));
  }
  if (method == 1 && !qd.crit) {
    // TOPSIS: the whole-GPU cluster kernel (nacs_rank.cu) on the context state
    nacs::RankManyArgs a = rank_many_args(ctx, o, qd, ctx->state.p, g.words(), 1);
    CK(nacs::launch_rank_many(a, ctx->num_sms, ctx->stream));
  } else {
    CK(nacs::launch_rank(g, o, ctx->state.p, qd, ctx->ahp_ws.p, ctx->w64.p, ctx->stats.p, ctx->stream));
  }
  if (!dev) {
    if (mask) CK(cudaMemcpyAsync(mask, qd.mask, g.n, cudaMemcpyDeviceToHost, ctx->stream));
    if (scores) CK(cudaMemcpyAsync(scores, qd.scores, 4 * (size_t)g.n, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(best, qd.best, 4, cudaMemcpyDeviceToHost, ctx->stream));
  }
  if (!(opt->flags & NACS_ASYNC)) {
    CK(cudaStreamSynchronize(ctx->stream));
    if ((st = finish_stats(ctx))) return st;
  }
  return NACS_OK;
}

#define NCK(call)                                                                   \
  do {                                                                              \
    ncclResult_t r_ = (call);                                                       \
    if (r_ != ncclSuccess) return fail(ctx, NACS_ENCCL, std::string(#call) + ": " + ncclGetErrorString(r_)); \
  } while (0)

// Sequential scheduling with the servers sharded over the ranks (k_sh_* kernels): the host
// drives each pod step (prepare, score own block, exchange keys, decide + commit) and reads
// the control word once per step.
nacs_status schedule_sharded(nacs_ctx* ctx, const Opt& o, const nacs::ReqsDev& Rd, const nacs::OutDev& Od, int R) {
  const Geo& g = ctx->g;
  const int world = ctx->world;
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  const size_t nW = (size_t)(g.n + 31) / 32, nEW = (size_t)(g.E + 31) / 32;
  const size_t b_gs = al(nacs::scratch_bytes()), b_bm = al(4 * nW), b_e = al(4 * nEW), b_ctl = al(16),
               b_kx = al(16 * (size_t)world), b_kv = al(8 * (size_t)world), b_ki = al(4 * (size_t)world);
  const bool ahp = o.method == NACS_AHP;
  size_t n2 = 1;
  while (n2 < (size_t)g.n) n2 <<= 1;
  const size_t b_ws = ahp ? al(nacs::ahp_workspace_bytes(g.n)) : 0, b_lv = ahp ? al(4 * 8 * n2) : 0,
               b_pp = ahp ? al(4 * 8 * (n2 + 2)) : 0, b_lvl = ahp ? al(4 * 4 * (size_t)g.n) : 0,
               b_f = ahp ? al(4 * 4 * n2) : 0, b_d = ahp ? al(4 * 8 * n2) : 0, b_K = ahp ? al(16) : 0;
  const int npart = std::max(1, std::min(256, (g.n + 1023) / 1024));
  const size_t b_facc = al(16 * 8), b_lsc = ahp ? al(4 * 5 * 4 * (n2 + 1)) : 0,
               b_kp = ahp ? al(2 * 8 * (size_t)npart) : 0, b_mt = ahp ? al(4 * nacs::AHP_MID_WARPS * 2 * 8) : 0;
  CK(ctx->sh_buf.reserve(b_gs + 2 * b_bm + b_e + b_ctl + b_kx + b_kv + b_ki + b_facc + b_ws + 2 * b_lv + 2 * b_pp +
                         b_lvl + 2 * b_f + 2 * b_d + b_K + b_lsc + b_kp + b_mt));
  CK(ctx->sh_ctl.reserve(16));
  CK(ctx->ulog.reserve(nacs::ULOG_CAP));
  CK(ctx->misc.reserve(8));
  unsigned char* p = ctx->sh_buf.p;
  nacs::ShardDev d;
  d.gs = reinterpret_cast<nacs::Scratch*>(p); p += b_gs;
  d.maskw = reinterpret_cast<unsigned*>(p); p += b_bm;
  d.special = reinterpret_cast<unsigned*>(p); p += b_bm;
  d.edgebad = reinterpret_cast<unsigned*>(p); p += b_e;
  d.ctl = reinterpret_cast<int*>(p); p += b_ctl;
  d.kx = reinterpret_cast<unsigned long long*>(p); p += b_kx;
  d.kxv = reinterpret_cast<double*>(p); p += b_kv;
  d.kxi = reinterpret_cast<int*>(p); p += b_ki;
  d.facc = reinterpret_cast<unsigned long long*>(p); p += b_facc;
  d.ahp_ws = nullptr;
  d.lvmC = d.lvwC = nullptr;
  d.paC = d.pbC = nullptr;
  d.lvlC = nullptr;
  d.wq = d.l2q = nullptr;
  d.wq64 = d.l2q64 = nullptr;
  d.Kc = nullptr;
  d.lvscr = nullptr;
  d.kpart = nullptr;
  d.midtot = nullptr;
  if (ahp) {
    d.ahp_ws = p; p += b_ws;
    d.lvmC = reinterpret_cast<float2*>(p); p += b_lv;
    d.lvwC = reinterpret_cast<float2*>(p); p += b_lv;
    d.paC = reinterpret_cast<double*>(p); p += b_pp;
    d.pbC = reinterpret_cast<double*>(p); p += b_pp;
    d.lvlC = reinterpret_cast<int*>(p); p += b_lvl;
    d.wq = reinterpret_cast<float*>(p); p += b_f;
    d.l2q = reinterpret_cast<float*>(p); p += b_f;
    d.wq64 = reinterpret_cast<double*>(p); p += b_d;
    d.l2q64 = reinterpret_cast<double*>(p); p += b_d;
    d.Kc = reinterpret_cast<int*>(p); p += b_K;
    d.lvscr = reinterpret_cast<int*>(p); p += b_lsc;
    d.kpart = reinterpret_cast<unsigned long long*>(p); p += b_kp;
    d.midtot = reinterpret_cast<double*>(p); p += b_mt;
  }
  d.npart = npart;
  d.ulog = ctx->ulog.p;
  d.stats = ctx->stats.p;
  CK(cudaMemsetAsync(d.maskw, 0, 2 * b_bm + b_e, ctx->stream));
  CK(cudaMemsetAsync(d.facc, 0, b_facc, ctx->stream));  // [14]: no presorted-order update pending
  int* ctl = reinterpret_cast<int*>(ctx->sh_ctl.p);
  // this process's shards: all of them in loopback, its own rank otherwise
  const int s_lo = ctx->loopback ? 0 : ctx->rank, s_hi = ctx->loopback ? world : ctx->rank + 1;
  auto lo_of = [&](int q) { return (int)((long long)g.n * q / world); };
  const bool dbg = getenv("NACS_DEBUG_SHARD") != nullptr;
  for (int r = 0; r < R; ++r) {
    CK(nacs::launch_sh_begin(g, o, ctx->state.p, Rd, Od, r, d, ctx->stream));
    for (long it = 0;; ++it) {
      CK(cudaMemcpyAsync(ctl, d.ctl, 16, cudaMemcpyDeviceToHost, ctx->stream));
      CK(cudaStreamSynchronize(ctx->stream));
      const int phase = ctl[0];
      if (dbg) fprintf(stderr, "[shard] r=%d it=%ld phase=%d pod=%d best=%d fail=%d\n", r, it, phase, ctl[1], ctl[2],
                       ctl[3]);
      if (phase == 0) {  // PH_DONE (AHP: an accepted request's touched servers into the presorted orders)
        if (ahp) CK(nacs::launch_presort_update(g, o, ctx->state.p, d, ctx->stream));
        break;
      }
      if (it > 4L * (g.n + 1) * (nacs::MAXC + 1))
        return fail(ctx, NACS_ECUDA, "sharded engine: pod loop did not finish (phase " + std::to_string(phase) + ")");
      if (ahp) {  // AHP: passes over this process's share of level pairs, sum-allreduce between
        // (loopback: one launch per logical rank, so the per-rank pair split runs as under NCCL)
        const bool f64 = phase == 3;
        if (!f64) CK(nacs::launch_sh_prep(g, o, ctx->state.p, Rd, Od, r, d, ctx->stream));
        for (int q = s_lo; q < s_hi; ++q)
          CK(nacs::launch_ahp_pass(1, f64, g, o, ctx->state.p, q, q + 1, world, d, ctx->num_sms, ctx->stream));
        if (ctx->comm) {
          if (f64) NCK(ncclAllReduce(d.wq64, d.wq64, 4 * n2, ncclFloat64, ncclSum, ctx->comm, ctx->stream));
          else NCK(ncclAllReduce(d.wq, d.wq, 4 * n2, ncclFloat32, ncclSum, ctx->comm, ctx->stream));
        }
        CK(nacs::launch_ahp_mid(f64, g, o, ctx->state.p, d, ctx->stream));
        for (int q = s_lo; q < s_hi; ++q)
          CK(nacs::launch_ahp_pass(2, f64, g, o, ctx->state.p, q, q + 1, world, d, ctx->num_sms, ctx->stream));
        if (ctx->comm) {
          if (f64) NCK(ncclAllReduce(d.l2q64, d.l2q64, 4 * n2, ncclFloat64, ncclSum, ctx->comm, ctx->stream));
          else NCK(ncclAllReduce(d.l2q, d.l2q, 4 * n2, ncclFloat32, ncclSum, ctx->comm, ctx->stream));
        }
        CK(nacs::launch_ahp_decide(f64, g, o, ctx->state.p, Rd, Od, r, d, ctx->stream));
        continue;
      }
      if (phase == 3) {       // PH_FP64: re-decide the near tie in FP64
        for (int q = s_lo; q < s_hi; ++q)
          CK(nacs::launch_sh_fp64(g, o, ctx->state.p, lo_of(q), lo_of(q + 1), q, d, ctx->stream));
        if (ctx->comm) {
          NCK(ncclAllGather(d.kxv + ctx->rank, d.kxv, 1, ncclFloat64, ctx->comm, ctx->stream));
          NCK(ncclAllGather(d.kxi + ctx->rank, d.kxi, 1, ncclInt32, ctx->comm, ctx->stream));
        }
        if (dbg) {
          std::vector<int> ki(world);
          std::vector<double> kv(world);
          std::vector<unsigned long long> kk(2 * world);
          CK(cudaMemcpyAsync(ki.data(), d.kxi, 4 * world, cudaMemcpyDeviceToHost, ctx->stream));
          CK(cudaMemcpyAsync(kv.data(), d.kxv, 8 * world, cudaMemcpyDeviceToHost, ctx->stream));
          CK(cudaMemcpyAsync(kk.data(), d.kx, 16 * world, cudaMemcpyDeviceToHost, ctx->stream));
          CK(cudaStreamSynchronize(ctx->stream));
          for (int q = 0; q < world; ++q)
            fprintf(stderr, "  fp64 slot %d: %d %.17g keys %016llx %016llx\n", q, ki[q], kv[q], kk[2 * q], kk[2 * q + 1]);
        }
        CK(nacs::launch_sh_decide64(g, o, ctx->state.p, Rd, Od, r, world, d, ctx->stream));
        continue;
      }
      CK(nacs::launch_sh_prep(g, o, ctx->state.p, Rd, Od, r, d, ctx->stream));
      for (int q = s_lo; q < s_hi; ++q)
        CK(nacs::launch_sh_score(g, o, ctx->state.p, lo_of(q), lo_of(q + 1), q, d, ctx->stream));
      if (ctx->comm) NCK(ncclAllGather(d.kx + 2 * ctx->rank, d.kx, 2, ncclUint64, ctx->comm, ctx->stream));
      CK(nacs::launch_sh_decide(g, o, ctx->state.p, Rd, Od, r, world, d, ctx->stream));
    }
  }
  return NACS_OK;
}

}  // namespace

extern "C" {

nacs_status nacs_nccl_unique_id(void* out) {
  if (!out) return NACS_EINVAL;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return NACS_ENCCL;
  std::memcpy(out, &id, sizeof(id));
  return NACS_OK;
}

nacs_status nacs_create_sharded(nacs_ctx** out, int device, void* cuda_stream, const void* nccl_unique_id, int rank,
                                int world) {
  if (!out || world < 1 || rank < 0 || rank >= world) return NACS_EINVAL;
  nacs_status st = nacs_create(out, device, cuda_stream);
  if (st) return st;
  nacs_ctx* ctx = *out;
  ctx->rank = rank;
  ctx->world = world;
  if (nccl_unique_id) {
    ncclUniqueId id;
    std::memcpy(&id, nccl_unique_id, sizeof(id));
    if (ncclCommInitRank(&ctx->comm, world, id, rank) != ncclSuccess) {
      nacs_destroy(ctx);
      *out = nullptr;
      return NACS_ENCCL;
    }
  } else if (world > 1) {
    ctx->loopback = true;
  }
  return NACS_OK;
}

nacs_status nacs_create(nacs_ctx** out, int device, void* cuda_stream) {
  if (!out) return NACS_EINVAL;
  *out = nullptr;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    cudaGetLastError();
    return NACS_ECUDA;
  }
  if (device < 0 || device >= count) return NACS_EINVAL;
  nacs_ctx* ctx = new nacs_ctx();
  ctx->device = device;
  const char* env = getenv("NACS_CTA_ONLY");
  ctx->cta_only = env && env[0] == '1';
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (e == cudaSuccess) ctx->stream = static_cast<cudaStream_t>(cuda_stream);
  if (e != cudaSuccess) {
    delete ctx;
    cudaGetLastError();
    return NACS_ECUDA;
  }
  *out = ctx;
  return NACS_OK;
}

void nacs_destroy(nacs_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  ctx->state.release();
  ctx->req_in.release();
  ctx->req_out.release();
  ctx->ulog.release();
  ctx->wlog.release();
  ctx->wlay.release();
  ctx->deferred.release();
  ctx->w64.release();
  ctx->ahp_ws.release();
  ctx->ahp_glob.release();
  ctx->seqc.release();
  ctx->misc.release();
  ctx->mask.release();
  ctx->scores.release();
  ctx->stats.release();
  ctx->pin_in.release();
  ctx->pin_out.release();
  ctx->sh_buf.release();
  ctx->sh_ctl.release();
  ctx->g_off.release();
  ctx->g_adj.release();
  ctx->g_adj16.release();
  ctx->g_scratch.release();
  ctx->g_io.release();
  ctx->g_out.release();
  ctx->g_ws.release();
  ctx->crit.release();
  ctx->many.release();
  ctx->many_mask.release();
  ctx->many_scores.release();
  ctx->rel_delta.release();
  ctx->sim_buf.release();
  ctx->sim_pin.release();
  if (ctx->comm) ncclCommDestroy(ctx->comm);
  if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

nacs_status nacs_load_topology(nacs_ctx* ctx, const nacs_topology* t) {
  NvtxRange nvtx_range_("nacs_load_topology");
  if (!ctx) return NACS_EINVAL;
  ctx->err.clear();
  if (!t) return fail(ctx, NACS_EINVAL, "topology: NULL");
  std::string m;
  if (t->k < 2 || t->k % 2) m += "k must be even and >= 2; ";
  if (t->cpu_cap <= 0 || t->ram_cap <= 0 || t->link_cap <= 0) m += "capacities must be > 0; ";
  if (!m.empty()) return fail(ctx, NACS_EINVAL, m);
  if (t->k > NACS_MAX_K) return fail(ctx, NACS_ETOOBIG, "k > NACS_MAX_K (64)");
  if (t->cpu_cap > NACS_MAX_CAP || t->ram_cap > NACS_MAX_CAP || t->link_cap > NACS_MAX_CAP)
    return fail(ctx, NACS_ETOOBIG, "a capacity exceeds NACS_MAX_CAP (2^23-1)");
  Geo g;
  g.k = t->k;
  g.h = t->k / 2;
  g.n = t->k * t->k * t->k / 4;
  g.E = t->k * t->k / 2;
  g.L = 3 * g.n;
  g.cpu_cap = t->cpu_cap;
  g.ram_cap = t->ram_cap;
  g.link_cap = t->link_cap;
  g.magic_h = g.h == 1 ? 0u : (unsigned)((((unsigned long long)1 << 32) + g.h - 1) / g.h);  // div_h
  std::vector<int> h((size_t)g.words());
  int n = g.n;
  int bad_cpu = 0, bad_ram = 0, bad_act = 0, bad_link = 0;
  for (int u = 0; u < n; ++u) {
    int c = t->cpu_res ? t->cpu_res[u] : g.cpu_cap;
    int r = t->ram_res ? t->ram_res[u] : g.ram_cap;
    if (c < 0 || c > g.cpu_cap) ++bad_cpu;
    if (r < 0 || r > g.ram_cap) ++bad_ram;
    int a;
    if (t->active) {
      a = t->active[u];
      if (a > 1) ++bad_act;
    } else {
      a = (c < g.cpu_cap || r < g.ram_cap) ? 1 : 0;
    }
    h[u] = c;
    h[n + u] = r;
    h[2 * n + u] = a;
  }
  for (int l = 0; l < g.L; ++l) {
    int b = t->link_res ? t->link_res[l] : g.link_cap;
    if (b < 0 || b > g.link_cap) ++bad_link;
    h[3 * n + l] = b;
  }
  if (bad_cpu) m += std::to_string(bad_cpu) + " cpu_res outside [0, cpu_cap]; ";
  if (bad_ram) m += std::to_string(bad_ram) + " ram_res outside [0, ram_cap]; ";
  if (bad_act) m += std::to_string(bad_act) + " active not 0/1; ";
  if (bad_link) m += std::to_string(bad_link) + " link_res outside [0, link_cap]; ";
  if (!m.empty()) return fail(ctx, NACS_EINVAL, m);
  CK(cudaSetDevice(ctx->device));
  CK(ctx->state.reserve(h.size()));
  CK(cudaMemcpyAsync(ctx->state.p, h.data(), h.size() * 4, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->g = g;
  ctx->has_topo = true;
  return NACS_OK;
}

nacs_status nacs_read_topology(nacs_ctx* ctx, int32_t* cpu_res, int32_t* ram_res, uint8_t* active,
                               int32_t* link_res) {
  if (!ctx) return NACS_EINVAL;
  ctx->err.clear();
  if (!ctx->has_topo) return fail(ctx, NACS_ENOTOPO, "no topology loaded");
  CK(cudaSetDevice(ctx->device));
  const Geo& g = ctx->g;
  std::vector<int> h((size_t)g.words());
  CK(cudaMemcpyAsync(h.data(), ctx->state.p, h.size() * 4, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  int n = g.n;
  for (int u = 0; u < n; ++u) {
    if (cpu_res) cpu_res[u] = h[u];
    if (ram_res) ram_res[u] = h[n + u];
    if (active) active[u] = (uint8_t)h[2 * n + u];
  }
  if (link_res) std::memcpy(link_res, h.data() + 3 * n, (size_t)g.L * 4);
  return NACS_OK;
}

nacs_status nacs_rank_ahp(nacs_ctx* ctx, const nacs_options* opt, const nacs_pod_query* q, uint8_t* mask,
                          float* scores, int32_t* best) {
  NvtxRange nvtx_range_("nacs_rank_ahp");
  return rank_impl(ctx, opt, q, mask, scores, best, 0);
}

nacs_status nacs_rank_topsis(nacs_ctx* ctx, const nacs_options* opt, const nacs_pod_query* q, uint8_t* mask,
                             float* scores, int32_t* best) {
  NvtxRange nvtx_range_("nacs_rank_topsis");
  return rank_impl(ctx, opt, q, mask, scores, best, 1);
}

nacs_status nacs_rank_topsis_many(nacs_ctx* ctx, const nacs_options* opt, const nacs_pod_query* q, int32_t n_states,
                                  const int32_t* states, int64_t state_stride, uint8_t* mask, float* scores,
                                  int32_t* best) {
  NvtxRange nvtx_range_("nacs_rank_topsis_many");
  nacs_status st = begin_call(ctx);
  if (st) return st;
  Opt o;
  if ((st = check_options(ctx, opt, &o))) return st;
  if (o.method != NACS_TOPSIS) return fail(ctx, NACS_EINVAL, "nacs_rank_topsis_many: options.method must be NACS_TOPSIS");
  if (o.bw_logical) return fail(ctx, NACS_EINVAL, "nacs_rank_topsis_many: bw_criterion must be NACS_BW_ACCESS");
  if (ctx->world > 1 || ctx->comm) return fail(ctx, NACS_EINVAL, "nacs_rank_topsis_many: not on server-sharded contexts");
  if (!q || n_states < 0 || (n_states > 0 && (!states || !best)))
    return fail(ctx, NACS_EINVAL, "nacs_rank_topsis_many: query/states/best NULL or n_states < 0");
  const Geo& g = ctx->g;
  if (state_stride < g.words())
    return fail(ctx, NACS_EINVAL, "nacs_rank_topsis_many: state_stride < 3n + L words");
  if (nacs::rank_many_cluster(g) > 16) return fail(ctx, NACS_ETOOBIG, "nacs_rank_topsis_many: n > 65536");
  const bool dev = opt->flags & NACS_DEVICE_PTRS;
  nacs::QueryDev qd{};
  if ((st = query_device(ctx, q, dev, &qd))) return st;
  if (n_states == 0) return finish_stats(ctx);
  const size_t B = (size_t)n_states, n = (size_t)g.n;
  const int* d_states = states;
  long long stride = state_stride;
  if (!dev) {  // stage through device buffers (the product path is the device-pointer call)
    stride = g.words() + ((4 - g.words() % 4) % 4);
    CK(ctx->many.reserve(B * (size_t)stride + B + 4));
    CK(cudaMemcpy2DAsync(ctx->many.p, 4 * (size_t)stride, states, 4 * (size_t)state_stride, 4 * (size_t)g.words(), B,
                         cudaMemcpyHostToDevice, ctx->stream));
    d_states = ctx->many.p;
    if (mask) CK(ctx->many_mask.reserve(B * n));
    if (scores) CK(ctx->many_scores.reserve(B * n));
    qd.mask = mask ? ctx->many_mask.p : nullptr;
    qd.scores = scores ? ctx->many_scores.p : nullptr;
    qd.best = ctx->many.p + B * (size_t)stride;
  } else {
    if (((uintptr_t)scores % 16) || ((uintptr_t)mask % 4) || ((uintptr_t)states % 16) || ((uintptr_t)best % 4) ||
        (state_stride % 2))
      return fail(ctx, NACS_EINVAL,
                  "nacs_rank_topsis_many: device arrays must be aligned (states, scores 16 B; mask, best 4 B; "
                  "an even state_stride)");
    qd.mask = mask;
    qd.scores = scores;
    qd.best = best;
  }
  nacs::RankManyArgs a = rank_many_args(ctx, o, qd, d_states, stride, n_states);
  CK(nacs::launch_rank_many(a, ctx->num_sms, ctx->stream));
  if (!dev) {
    if (mask) CK(cudaMemcpyAsync(mask, qd.mask, B * n, cudaMemcpyDeviceToHost, ctx->stream));
    if (scores) CK(cudaMemcpyAsync(scores, qd.scores, 4 * B * n, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(best, qd.best, 4 * B, cudaMemcpyDeviceToHost, ctx->stream));
  }
  if (!(opt->flags & NACS_ASYNC)) {
    CK(cudaStreamSynchronize(ctx->stream));
    if ((st = finish_stats(ctx))) return st;
    if (ctx->last.invalid > 0)
      return fail(ctx, NACS_EINVAL, std::to_string(ctx->last.invalid) +
                                        " states hold a value outside [0, capacity] or f_u outside {0,1} (best = -2)");
  }
  return NACS_OK;
}

nacs_status nacs_schedule_batch(nacs_ctx* ctx, const nacs_options* opt, const nacs_requests* batch,
                                nacs_placements* out) {
  NvtxRange nvtx_range_("nacs_schedule_batch");
  nacs_status st = begin_call(ctx);
  if (st) return st;
  Opt o;
  if ((st = check_options(ctx, opt, &o))) return st;
  if (o.bw_logical) return fail(ctx, NACS_EINVAL, "options.bw_criterion = NACS_BW_LOGICAL: rank calls only");
  if ((st = check_placements(ctx, out))) return st;
  if (!batch || batch->n_requests < 0) return fail(ctx, NACS_EINVAL, "requests: NULL or n_requests < 0");
  const bool dev = opt->flags & NACS_DEVICE_PTRS;
  const Geo& g = ctx->g;
  if (!nacs::batch_smem_bytes(g, o.method))
    return fail(ctx, NACS_ETOOBIG, "snapshot does not fit in shared memory for nacs_schedule_batch");
  int R = batch->n_requests;
  if (R == 0) return finish_stats(ctx);
  nacs::ReqsDev Rd;
  nacs::OutDev Od;
  int C = 0, V = 0;
  static const bool timing = getenv("NACS_HOST_TIMING") != nullptr;
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto ms = [](std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) {
    return std::chrono::duration<double, std::milli>(b - a).count();
  };
  const auto t0 = now();
  auto t1 = t0, t2 = t0;
  if (!dev) {  // R24 validation of every request runs on the host while the kernels run
    if ((st = check_offsets_host(ctx, batch, &C, &V))) return st;
    t1 = now();
    if ((st = stage_requests(ctx, batch, C, V, &Rd))) return st;
    if ((st = mapped_outputs(ctx, R, C, V, &Od))) return st;
    t2 = now();
  } else {
    Rd = device_requests(batch);
    Od.status = out->status;
    Od.server = out->server_of_container;
    Od.cpu_a = out->cpu_alloc;
    Od.ram_a = out->ram_alloc;
    Od.bw_a = out->bw_alloc;
    Od.path = out->path_of_vlink;
  }
  int per_sm = 0;
  CK(nacs::batch_occupancy(g, o.method, &per_sm));
  if (per_sm <= 0) return fail(ctx, NACS_ETOOBIG, "batch kernel cannot be resident");
  int grid = ctx->num_sms * per_sm;
  if (grid > R) grid = R;
  CK(ctx->ulog.reserve((size_t)grid * nacs::ULOG_CAP));
  if (o.method == 0 || o.rank_once) CK(ctx->w64.reserve((size_t)grid * nacs::ahp_workspace_doubles(g.n)));
  unsigned char* ahp_g = nullptr;
  if (nacs::batch_ahp_global(g, o.method)) {
    const size_t per = (nacs::ahp_workspace_bytes(g.n) + 15) & ~(size_t)15;
    CK(ctx->ahp_glob.reserve((size_t)grid * per));
    ahp_g = ctx->ahp_glob.p;
  }
  CK(ctx->misc.reserve(8));
  CK(cudaMemsetAsync(ctx->misc.p, 0, 4 * sizeof(int), ctx->stream));
  const int warps = o.method == NACS_TOPSIS && !ctx->cta_only ? nacs::warp_kernel_warps(g) : 0;
  if (warps >= 4) {
    // fast path: warp per request; requests beyond its limits are deferred to k_batch
    int wgrid = ctx->num_sms;
    CK(ctx->wlog.reserve(nacs::warp_ulog_entries(wgrid, warps)));
    CK(ctx->wlay.reserve(nacs::warp_layout_ints(g)));
    CK(ctx->deferred.reserve(2 * (size_t)R));
    CK(nacs::launch_batch_warp(g, o, ctx->state.p, ctx->wlay.p, Rd, Od, ctx->wlog.p, ctx->misc.p, ctx->deferred.p + R,
                               ctx->deferred.p, ctx->misc.p + 2, ctx->stats.p, wgrid, warps, ctx->stream));
    CK(nacs::launch_batch(g, o, ctx->state.p, Rd, Od, ctx->ulog.p, ctx->w64.p, ahp_g, ctx->misc.p + 1, ctx->stats.p,
                          grid, ctx->stream, ctx->deferred.p, ctx->misc.p + 2));
  } else {
    CK(nacs::launch_batch(g, o, ctx->state.p, Rd, Od, ctx->ulog.p, ctx->w64.p, ahp_g, ctx->misc.p, ctx->stats.p, grid,
                          ctx->stream));
  }
  if (!dev) {
    const auto t3 = now();
    const nacs_status vst = validate_requests_host(ctx, batch);
    const auto t4 = now();
    CK(cudaStreamSynchronize(ctx->stream));
    const auto t5 = now();
    copy_mapped_outputs(ctx, R, C, V, out);
    if (timing)
      fprintf(stderr, "nacs host timing ms: offsets %.3f stage %.3f launch %.3f validate %.3f wait %.3f unstage %.3f\n",
              ms(t0, t1), ms(t1, t2), ms(t2, t3), ms(t3, t4), ms(t4, t5), ms(t5, now()));
    if (vst) {  // invalid requests carry status -1 in the outputs; the call reports them
      if (!(opt->flags & NACS_ASYNC)) finish_stats(ctx);
      return vst;
    }
  }
  if (!(opt->flags & NACS_ASYNC)) {
    CK(cudaStreamSynchronize(ctx->stream));
    if ((st = finish_stats(ctx))) return st;
    if (ctx->last.invalid > 0)
      return fail(ctx, NACS_EINVAL, std::to_string(ctx->last.invalid) + " invalid requests (status -1)");
  }
  return NACS_OK;
}

nacs_status nacs_schedule_request(nacs_ctx* ctx, const nacs_options* opt, const nacs_requests* reqs,
                                  nacs_placements* out) {
  NvtxRange nvtx_range_("nacs_schedule_request");
  nacs_status st = begin_call(ctx);
  if (st) return st;
  Opt o;
  if ((st = check_options(ctx, opt, &o))) return st;
  if (o.bw_logical) return fail(ctx, NACS_EINVAL, "options.bw_criterion = NACS_BW_LOGICAL: rank calls only");
  if ((st = check_placements(ctx, out))) return st;
  if (!reqs || reqs->n_requests < 0) return fail(ctx, NACS_EINVAL, "requests: NULL or n_requests < 0");
  const bool dev = opt->flags & NACS_DEVICE_PTRS;
  const bool async = opt->flags & NACS_ASYNC;
  const Geo& g = ctx->g;
  int R = reqs->n_requests;
  if (R == 0) return finish_stats(ctx);
  nacs::ReqsDev Rd;
  nacs::OutDev Od;
  int C = 0, V = 0;
  if (!dev) {
    if ((st = check_requests_host(ctx, reqs, &C, &V))) return st;
    if ((st = stage_requests(ctx, reqs, C, V, &Rd))) return st;
    if ((st = device_outputs(ctx, R, C, V, &Od))) return st;
  } else {
    Rd = device_requests(reqs);
    Od.status = out->status;
    Od.server = out->server_of_container;
    Od.cpu_a = out->cpu_alloc;
    Od.ram_a = out->ram_alloc;
    Od.bw_a = out->bw_alloc;
    Od.path = out->path_of_vlink;
    if (!async) {  // validate before touching the state: an error leaves it unchanged
      CK(nacs::launch_validate(Rd, Od.status, ctx->stats.p, ctx->stream));
      unsigned long long h[nacs::ST_N];
      CK(cudaMemcpyAsync(h, ctx->stats.p, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
      CK(cudaStreamSynchronize(ctx->stream));
      if (h[nacs::ST_INVALID])
        return fail(ctx, NACS_EINVAL, std::to_string(h[nacs::ST_INVALID]) + " invalid requests");
    }
  }
  // the sharded engine: server-sharded contexts, and (grid-wide level passes) AHP on big topologies
  if (o.rank_once && (ctx->world > 1 || ctx->comm))
    return fail(ctx, NACS_EINVAL, "options.rank_mode = NACS_RANK_ONCE is not available on server-sharded contexts");
  if (o.method >= NACS_BF && (ctx->world > 1 || ctx->comm))
    return fail(ctx, NACS_EINVAL, "BF / WF are not available on server-sharded contexts");
  if (ctx->comm_aborted)
    return fail(ctx, NACS_ENCCL, "the NCCL communicator of this context was aborted after an earlier error");
  if (ctx->world > 1 || ctx->comm || (o.method == NACS_AHP && g.n >= 4096 && !o.rank_once)) {
    if ((st = schedule_sharded(ctx, o, Rd, Od, R))) {
      // the other ranks may be waiting in this pod step's collective: abort the communicator so
      // that they fail instead of hanging, and refuse further sharded calls on this context
      if (ctx->comm) {
        ncclCommAbort(ctx->comm);
        ctx->comm = nullptr;
        ctx->comm_aborted = true;
      }
      return st;
    }
    if (!dev) {
      if ((st = unstage_outputs(ctx, R, C, V, out))) return st;
    }
    if (!async) {
      CK(cudaStreamSynchronize(ctx->stream));
      if ((st = finish_stats(ctx))) return st;
    }
    return NACS_OK;
  }
  CK(ctx->ulog.reserve(nacs::ULOG_CAP));
  const int seqc = o.method == NACS_TOPSIS && !o.rank_once ? nacs::seq_cluster_size(g) : 0;
  if (seqc > 0) {  // TOPSIS on a large DC: the whole request stream on one thread-block cluster
    CK(ctx->seqc.reserve(96));
    CK(nacs::launch_seq_cluster(g, o, ctx->state.p, Rd, Od, ctx->ulog.p, ctx->stats.p, ctx->seqc.p, seqc,
                                ctx->stream));
    if (!dev) {
      if ((st = unstage_outputs(ctx, R, C, V, out))) return st;
    }
    if (!async) {
      CK(cudaStreamSynchronize(ctx->stream));
      if ((st = finish_stats(ctx))) return st;
    }
    return NACS_OK;
  }
  if (o.method == 0) CK(ctx->ahp_ws.reserve(nacs::ahp_workspace_bytes(g.n) / 4 + 4));
  if (o.method == 0 || o.rank_once) CK(ctx->w64.reserve(nacs::ahp_workspace_doubles(g.n)));
  CK(nacs::launch_sequential(g, o, ctx->state.p, Rd, Od, ctx->ulog.p, ctx->ahp_ws.p, ctx->w64.p, ctx->stats.p,
                             ctx->stream));
  if (!dev) {
    if ((st = unstage_outputs(ctx, R, C, V, out))) return st;
  }
  if (!async) {
    CK(cudaStreamSynchronize(ctx->stream));
    if ((st = finish_stats(ctx))) return st;
  }
  return NACS_OK;
}

// ---------------------------------------------------------------------------------------
// Departures and the discrete-event simulator.
// ---------------------------------------------------------------------------------------
nacs_status nacs_release(nacs_ctx* ctx, uint32_t flags, const nacs_requests* reqs, const nacs_placements* pl) {
  NvtxRange nvtx_range_("nacs_release");
  nacs_status st = begin_call(ctx);
  if (st) return st;
  if (flags & ~(NACS_DEVICE_PTRS | NACS_ASYNC)) return fail(ctx, NACS_EINVAL, "flags: only NACS_DEVICE_PTRS | NACS_ASYNC");
  if ((st = check_placements(ctx, pl))) return st;
  if (!reqs) return fail(ctx, NACS_EINVAL, "requests: NULL");
  if (ctx->world > 1 || ctx->comm) return fail(ctx, NACS_EINVAL, "nacs_release is not available on server-sharded contexts");
  const Geo& g = ctx->g;
  const bool dev = flags & NACS_DEVICE_PTRS;
  const int R = reqs->n_requests;
  if (R < 0) return fail(ctx, NACS_EINVAL, "requests.n_requests < 0");
  if (R == 0) return finish_stats(ctx);
  nacs::ReqsDev Rd;
  nacs::OutDev Pd;
  if (dev) {
    Rd = device_requests(reqs);
    Pd.status = pl->status;
    Pd.server = pl->server_of_container;
    Pd.cpu_a = pl->cpu_alloc;
    Pd.ram_a = pl->ram_alloc;
    Pd.bw_a = pl->bw_alloc;
    Pd.path = pl->path_of_vlink;
  } else {
    int C = 0, V = 0;
    if ((st = check_offsets_host(ctx, reqs, &C, &V))) return st;
    if ((st = stage_requests(ctx, reqs, C, V, &Rd))) return st;
    if ((st = device_outputs(ctx, R, C, V, &Pd))) return st;
    CK(cudaMemcpyAsync(Pd.status, pl->status, (size_t)R * 4, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(Pd.server, pl->server_of_container, (size_t)C * 4, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(Pd.cpu_a, pl->cpu_alloc, (size_t)C * 4, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(Pd.ram_a, pl->ram_alloc, (size_t)C * 4, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(Pd.bw_a, pl->bw_alloc, (size_t)V * 4, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(Pd.path, pl->path_of_vlink, (size_t)V * 4, cudaMemcpyHostToDevice, ctx->stream));
  }
  CK(ctx->rel_delta.reserve((size_t)g.words()));
  CK(ctx->misc.reserve(8));
  CK(nacs::launch_release(g, ctx->state.p, Rd, Pd, nullptr, 0, ctx->rel_delta.p, ctx->misc.p, ctx->stream));
  if (!(flags & NACS_ASYNC)) {
    int bad = 0;
    CK(cudaMemcpyAsync(&bad, ctx->misc.p, 4, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if ((st = finish_stats(ctx))) return st;
    if (bad & 1) return fail(ctx, NACS_EINVAL, "placements: a server, path or allocation does not match the fat-tree");
    if (bad & 2) return fail(ctx, NACS_EINVAL, "release would raise a residual above its capacity (released twice?)");
  }
  return NACS_OK;
}

nacs_status nacs_simulate(nacs_ctx* ctx, const nacs_options* opt, const nacs_requests* reqs, const int32_t* arrival,
                          const int32_t* duration, const nacs_sim_config* cfg, nacs_placements* out,
                          nacs_sim_report* rep) {
  NvtxRange nvtx_range_("nacs_simulate");
  nacs_status st = begin_call(ctx);
  if (st) return st;
  Opt o;
  if ((st = check_options(ctx, opt, &o))) return st;
  if (o.bw_logical) return fail(ctx, NACS_EINVAL, "options.bw_criterion = NACS_BW_LOGICAL: rank calls only");
  if (opt->flags & (NACS_DEVICE_PTRS | NACS_ASYNC))
    return fail(ctx, NACS_EINVAL, "nacs_simulate takes host pointers and is synchronous");
  if (o.rank_once) return fail(ctx, NACS_EINVAL, "nacs_simulate: rank_mode must be NACS_RANK_PER_POD");
  if (ctx->world > 1 || ctx->comm) return fail(ctx, NACS_EINVAL, "nacs_simulate is not available on server-sharded contexts");
  if (!cfg || !rep || !arrival || !duration) return fail(ctx, NACS_EINVAL, "config/report/arrival/duration: NULL");
  if ((st = check_placements(ctx, out))) return st;
  if (!rep->start_tick || !rep->attempts || !rep->tick_servers || !rep->tick_links || !rep->tick_queue)
    return fail(ctx, NACS_EINVAL, "report arrays: NULL");
  if (cfg->max_ticks < 1) return fail(ctx, NACS_EINVAL, "config.max_ticks < 1");
  if (cfg->hol_blocking != 0 && cfg->hol_blocking != 1) return fail(ctx, NACS_EINVAL, "config.hol_blocking not 0/1");
  int C = 0, V = 0;
  if ((st = check_requests_host(ctx, reqs, &C, &V))) return st;
  const int R = reqs->n_requests;
  for (int r = 0; r < R; ++r)
    if (arrival[r] < 0 || duration[r] < 1)
      return fail(ctx, NACS_EINVAL, "request " + std::to_string(r) + ": arrival < 0 or duration < 1");
  const Geo& g = ctx->g;
  const auto t_start = std::chrono::steady_clock::now();
  nacs::ReqsDev Rd;
  nacs::OutDev Od;
  if ((st = stage_requests(ctx, reqs, C, V, &Rd))) return st;
  if ((st = device_outputs(ctx, R, C, V, &Od))) return st;
  // requests never offered keep status 0, mappings -1, allocations 0
  CK(cudaMemsetAsync(Od.status, 0, sizeof(int) * (size_t)R, ctx->stream));
  CK(cudaMemsetAsync(Od.server, 0xFF, sizeof(int) * (size_t)C, ctx->stream));
  CK(cudaMemsetAsync(Od.cpu_a, 0, sizeof(int) * 2 * (size_t)C + sizeof(int) * (size_t)V, ctx->stream));
  CK(cudaMemsetAsync(Od.path, 0xFF, sizeof(int) * (size_t)V, ctx->stream));
  CK(ctx->ulog.reserve(nacs::ULOG_CAP));
  if (o.method == 0) CK(ctx->ahp_ws.reserve(nacs::ahp_workspace_bytes(g.n) / 4 + 4));
  if (o.method == 0) CK(ctx->w64.reserve(nacs::ahp_workspace_doubles(g.n)));
  // the whole event loop runs on the device in one launch (k_simulate)
  const int T = cfg->max_ticks;
  std::vector<int> order(R);
  for (int r = 0; r < R; ++r) order[r] = r;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return arrival[a] < arrival[b]; });
  // device: order | arrival | duration | start | attempts | qbuf | qtmp | run [R each] | ticks [3T] |
  // head [T] | totals
  CK(ctx->sim_buf.reserve(8 * (size_t)R + 4 * (size_t)T + 8));
  int* d = ctx->sim_buf.p;
  nacs::SimDev S;
  S.order = d;
  S.arrival = d + R;
  S.duration = d + 2 * (size_t)R;
  S.start = d + 3 * (size_t)R;
  S.attempts = d + 4 * (size_t)R;
  S.qbuf = d + 5 * (size_t)R;
  S.qtmp = d + 6 * (size_t)R;
  S.run = d + 7 * (size_t)R;
  S.ticks = d + 8 * (size_t)R;
  S.head = d + 8 * (size_t)R + 3 * (size_t)T;
  S.totals = reinterpret_cast<long long*>(d + ((8 * (size_t)R + 4 * (size_t)T + 1) & ~(size_t)1));
  S.max_ticks = T;
  S.hol = cfg->hol_blocking;
  CK(cudaMemcpyAsync(d, order.data(), (size_t)R * 4, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(d + R, arrival, (size_t)R * 4, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(d + 2 * (size_t)R, duration, (size_t)R * 4, cudaMemcpyHostToDevice, ctx->stream));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, ctx->stream));
  CK(nacs::launch_simulate(g, o, ctx->state.p, Rd, Od, ctx->ulog.p, ctx->ahp_ws.p, ctx->w64.p, ctx->stats.p, S,
                           ctx->stream));
  CK(cudaEventRecord(e1, ctx->stream));
  if ((st = unstage_outputs(ctx, R, C, V, out))) return st;
  long long tot[3];
  CK(cudaMemcpyAsync(tot, S.totals, sizeof(tot), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(rep->start_tick, S.start, (size_t)R * 4, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(rep->attempts, S.attempts, (size_t)R * 4, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  const int t = (int)tot[0];
  std::vector<int> ticks(3 * (size_t)t + 1);
  if (t) CK(cudaMemcpy(ticks.data(), S.ticks, 3 * (size_t)t * 4, cudaMemcpyDeviceToHost));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  for (int r = 0; r < R; ++r)
    if (rep->start_tick[r] < 0) out->status[r] = 0;
  for (int i = 0; i < t; ++i) {
    rep->tick_servers[i] = ticks[3 * i];
    rep->tick_links[i] = ticks[3 * i + 1];
    rep->tick_queue[i] = ticks[3 * i + 2];
  }
  rep->events = t;
  rep->attempts_total = tot[1];
  rep->accepted = tot[2];
  rep->sched_seconds = ms / 1e3;
  rep->wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
  return finish_stats(ctx);
}

// ---------------------------------------------------------------------------------------
// General topology: nacs_load_graph, nacs_widest_paths,
// nacs_logical_bandwidth.  The host builds the CSR layout once per graph; the modified
// Dijkstra runs in nacs_paths.cu.
// ---------------------------------------------------------------------------------------
static nacs::GraphDev graph_dev(nacs_ctx* ctx) {
  nacs::GraphDev G;
  G.V = ctx->gV;
  G.ns = ctx->gns;
  G.n_adj = 2 * ctx->gL;
  G.off = ctx->g_off.p;
  G.adj = ctx->g_adj.p;
  G.adj16 = ctx->g_packed ? ctx->g_adj16.p : nullptr;
  return G;
}

nacs_status nacs_load_graph(nacs_ctx* ctx, const nacs_graph* gr) {
  NvtxRange nvtx_range_("nacs_load_graph");
  if (!ctx) return NACS_EINVAL;
  ctx->err.clear();
  if (!gr) return fail(ctx, NACS_EINVAL, "graph: NULL");
  std::string m;
  const int V = gr->n_vertices, ns = gr->n_servers, nl = gr->n_links;
  if (V < 2) m += "n_vertices must be >= 2; ";
  if (ns < 1 || ns > V) m += "n_servers out of 1..n_vertices; ";
  if (nl < 0) m += "n_links < 0; ";
  if (nl > 0 && (!gr->link_u || !gr->link_v || !gr->link_res)) m += "link arrays NULL; ";
  if (!m.empty()) return fail(ctx, NACS_EINVAL, m);
  if (V > NACS_MAX_GRAPH_VERTICES || nl > NACS_MAX_GRAPH_LINKS)
    return fail(ctx, NACS_ETOOBIG, "graph exceeds NACS_MAX_GRAPH_VERTICES / NACS_MAX_GRAPH_LINKS");
  int bad_end = 0, bad_loop = 0, bad_res = 0;
  std::vector<int> deg((size_t)V + 1, 0);
  for (int l = 0; l < nl; ++l) {
    const int a = gr->link_u[l], b = gr->link_v[l], r = gr->link_res[l];
    if (a < 0 || a >= V || b < 0 || b >= V) { ++bad_end; continue; }
    if (a == b) ++bad_loop;
    if (r < 0 || r > NACS_MAX_CAP) ++bad_res;
    ++deg[a];
    ++deg[b];
  }
  if (bad_end) m += std::to_string(bad_end) + " link endpoints out of range; ";
  if (bad_loop) m += std::to_string(bad_loop) + " self-loops; ";
  if (bad_res) m += std::to_string(bad_res) + " link_res outside [0, NACS_MAX_CAP]; ";
  if (!m.empty()) return fail(ctx, NACS_EINVAL, m);
  std::vector<int> off((size_t)V + 1, 0);
  for (int v = 0; v < V; ++v) off[v + 1] = off[v] + deg[v];
  std::vector<int> at(off.begin(), off.end() - 1);
  std::vector<int2> adj((size_t)2 * nl + 1);
  int max_res = 0;
  for (int l = 0; l < nl; ++l) {
    const int a = gr->link_u[l], b = gr->link_v[l], r = gr->link_res[l];
    adj[at[a]++] = make_int2(b, r);
    adj[at[b]++] = make_int2(a, r);
    max_res = std::max(max_res, r);
  }
  // packed 4-byte entries for the shared-memory layout (nacs_paths.cu)
  const bool packed = V <= 65536 && max_res <= 65535;
  std::vector<unsigned> adj16;
  if (packed) {
    adj16.resize(adj.size());
    for (size_t j = 0; j < adj.size(); ++j) adj16[j] = (unsigned)adj[j].x | ((unsigned)adj[j].y << 16);
  }
  CK(cudaSetDevice(ctx->device));
  CK(ctx->g_off.reserve(off.size()));
  CK(ctx->g_adj.reserve(adj.size()));
  CK(cudaMemcpyAsync(ctx->g_off.p, off.data(), off.size() * 4, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ctx->g_adj.p, adj.data(), adj.size() * sizeof(int2), cudaMemcpyHostToDevice, ctx->stream));
  if (packed) {
    CK(ctx->g_adj16.reserve(adj16.size()));
    CK(cudaMemcpyAsync(ctx->g_adj16.p, adj16.data(), adj16.size() * 4, cudaMemcpyHostToDevice, ctx->stream));
  }
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->gV = V;
  ctx->gns = ns;
  ctx->gL = nl;
  ctx->g_packed = packed;
  ctx->has_graph = true;
  const nacs::PathLaunch c = nacs::path_launch_config(graph_dev(ctx), ctx->num_sms);
  if (c.global_bytes) CK(ctx->g_scratch.reserve(c.global_bytes / 4 + 1));
  return NACS_OK;
}

static nacs_status begin_graph_call(nacs_ctx* ctx, uint32_t flags) {
  if (!ctx) return NACS_EINVAL;
  ctx->err.clear();
  CK(cudaSetDevice(ctx->device));
  if (!ctx->has_graph) return fail(ctx, NACS_ENOTOPO, "no graph loaded (nacs_load_graph)");
  if (flags & ~(NACS_DEVICE_PTRS | NACS_ASYNC)) return fail(ctx, NACS_EINVAL, "flags: only NACS_DEVICE_PTRS | NACS_ASYNC");
  CK(ctx->stats.reserve(nacs::ST_N));
  CK(cudaMemsetAsync(ctx->stats.p, 0, sizeof(unsigned long long) * nacs::ST_N, ctx->stream));
  ctx->stats_pending = true;
  return NACS_OK;
}


nacs_status nacs_widest_paths(nacs_ctx* ctx, const nacs_path_query* q, uint32_t flags, int32_t* bottleneck,
                              int32_t* hops, int32_t* path, int32_t max_hops) {
  NvtxRange nvtx_range_("nacs_widest_paths");
  nacs_status st = begin_graph_call(ctx, flags);
  if (st) return st;
  if (!q || !bottleneck || !hops) return fail(ctx, NACS_EINVAL, "query/bottleneck/hops: NULL");
  const int nq = q->n_queries;
  std::string m;
  if (nq < 0) m += "n_queries < 0; ";
  if (nq > 0 && (!q->src || !q->dst || !q->demand)) m += "query arrays NULL; ";
  if (path && max_hops < 0) m += "max_hops < 0; ";
  if (!m.empty()) return fail(ctx, NACS_EINVAL, m);
  const bool dev = flags & NACS_DEVICE_PTRS;
  const int V = ctx->gV;
  const size_t prow = path ? (size_t)max_hops + 1 : 0;
  if (!dev) {
    int bad = 0, first = -1;
    for (int i = 0; i < nq; ++i) {
      const int s = q->src[i], t = q->dst[i], d = q->demand[i];
      if (s < 0 || s >= V || t < 0 || t >= V || s == t || d < 0 || d > NACS_MAX_CAP) {
        if (first < 0) first = i;
        ++bad;
      }
    }
    if (bad)
      return fail(ctx, NACS_EINVAL, std::to_string(bad) + " invalid queries (endpoint out of range, src == dst or demand "
                                    "outside [0, NACS_MAX_CAP]), first at " + std::to_string(first));
  }
  if (nq == 0) return finish_stats(ctx);
  const nacs::GraphDev G = graph_dev(ctx);
  const nacs::PathLaunch c = nacs::path_launch_config(G, ctx->num_sms);
  if (c.global_bytes) CK(ctx->g_scratch.reserve(c.global_bytes / 4 + 1));
  const int *dsrc, *ddst, *ddem;
  int *dbn, *dhops, *dpath;
  if (dev) {
    dsrc = q->src;
    ddst = q->dst;
    ddem = q->demand;
    dbn = bottleneck;
    dhops = hops;
    dpath = path;
  } else {
    const size_t in = 3 * (size_t)nq, out = 2 * (size_t)nq + (size_t)nq * prow;
    CK(ctx->g_io.reserve(in + out));
    CK(ctx->pin_in.reserve(in * 4));
    CK(ctx->pin_out.reserve(out * 4));
    int* hin = reinterpret_cast<int*>(ctx->pin_in.p);
    parallel_copies({{hin, q->src, (size_t)nq * 4}, {hin + nq, q->dst, (size_t)nq * 4},
                     {hin + 2 * (size_t)nq, q->demand, (size_t)nq * 4}});
    CK(cudaMemcpyAsync(ctx->g_io.p, hin, in * 4, cudaMemcpyHostToDevice, ctx->stream));
    dsrc = ctx->g_io.p;
    ddst = dsrc + nq;
    ddem = dsrc + 2 * (size_t)nq;
    dbn = ctx->g_io.p + in;
    dhops = dbn + nq;
    dpath = path ? dhops + nq : nullptr;
  }
  CK(ctx->g_ws.reserve(nacs::path_group_ints(V, nq)));
  CK(nacs::launch_paths(G, c, nq, dsrc, ddst, ddem, dbn, dhops, dpath, max_hops, ctx->g_ws.p, ctx->g_scratch.p,
                        ctx->stats.p, ctx->stream));
  if (!dev) {
    const size_t out = 2 * (size_t)nq + (size_t)nq * prow;
    int* hout = reinterpret_cast<int*>(ctx->pin_out.p);
    CK(cudaMemcpyAsync(hout, dbn, out * 4, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    std::vector<CopyJob> jobs{{bottleneck, hout, (size_t)nq * 4}, {hops, hout + nq, (size_t)nq * 4}};
    if (path) jobs.push_back({path, hout + 2 * (size_t)nq, (size_t)nq * prow * 4});
    parallel_copies(jobs);
  }
  if (!(flags & NACS_ASYNC)) {
    CK(cudaStreamSynchronize(ctx->stream));
    if ((st = finish_stats(ctx))) return st;
    if (dev && ctx->last.invalid)
      return fail(ctx, NACS_EINVAL, std::to_string(ctx->last.invalid) + " invalid queries (hops = -2)");
  }
  return NACS_OK;
}

nacs_status nacs_logical_bandwidth(nacs_ctx* ctx, uint32_t flags, int64_t* out) {
  NvtxRange nvtx_range_("nacs_logical_bandwidth");
  nacs_status st = begin_graph_call(ctx, flags);
  if (st) return st;
  if (!out) return fail(ctx, NACS_EINVAL, "out: NULL");
  const bool dev = flags & NACS_DEVICE_PTRS;
  const nacs::GraphDev G = graph_dev(ctx);
  const nacs::PathLaunch c = nacs::path_launch_config(G, ctx->num_sms);
  if (c.global_bytes) CK(ctx->g_scratch.reserve(c.global_bytes / 4 + 1));
  long long* dout = reinterpret_cast<long long*>(out);
  if (!dev) {
    CK(ctx->g_out.reserve(ctx->gns));
    dout = ctx->g_out.p;
  }
  CK(nacs::launch_logical_bw(G, c, dout, ctx->g_scratch.p, ctx->stats.p, ctx->stream));
  if (!dev) CK(cudaMemcpyAsync(out, dout, (size_t)ctx->gns * 8, cudaMemcpyDeviceToHost, ctx->stream));
  if (!(flags & NACS_ASYNC)) {
    CK(cudaStreamSynchronize(ctx->stream));
    if ((st = finish_stats(ctx))) return st;
  }
  return NACS_OK;
}

nacs_status nacs_last_stats(nacs_ctx* ctx, nacs_stats* out) {
  if (!ctx || !out) return NACS_EINVAL;
  nacs_status st = finish_stats(ctx);
  if (st) return st;
  *out = ctx->last;
  return NACS_OK;
}

const char* nacs_last_error(const nacs_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

}  // extern "C"
