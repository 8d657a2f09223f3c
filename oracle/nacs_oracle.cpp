// nacs_oracle.cpp — TEST INFRASTRUCTURE ONLY.
//
// A plain, slow, double-precision CPU implementation of the per-pod ranking and
// greedy placement of arXiv 1909.07673 ("Network-Aware Container Scheduling in
// Multi-Tenant Data Center", §V), written from the paper and the
// readings R1-R24 listed in DESIGN.md.  It exists only to check the CUDA path:
// only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
// arm may load it.  It shares no code, header, table or constant with
// paper_1909_07673_b200/ (the product), and the product never loads it.
//
// Every function follows the paper's order of operations with no blocking,
// fusion or reordering.  Citations: "P:n" = PAPER.md line n.
//
// Units (reading R5): CPU in millicores, RAM in MiB, bandwidth in Mbps, all
// integers; the residual state is integer and every score is a double.
//
// Build: g++ -O2 -std=c++17 -fopenmp -shared -fPIC (no fast-math).

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <vector>

namespace {

// ---------------------------------------------------------------------------
// DC model G^s(N^s, E^s) as a k-ary fat-tree (§II-A, §IV-B1).
// Servers u = 0..n-1; edge switch of u = u / h; pod of edge switch e = e / h.
// Physical links, canonical order: access[n] | edge-agg[E][h] | agg-core[k][h][h].
// ---------------------------------------------------------------------------
struct DC {
  int k = 0, h = 0, n = 0, E = 0, L = 0;
  long cpu_cap = 0, ram_cap = 0, link_cap = 0;
  std::vector<long> cpu, ram;   // residual c^s_u[r]
  std::vector<int> active;      // f_u (T2 P:150)
  std::vector<long> link;       // residual bandwidth per physical link

  int edge_of(int u) const { return u / h; }
  int pod_of_edge(int e) const { return e / h; }
  int access(int u) const { return u; }
  int ea(int e, int a) const { return n + e * h + a; }
  int ac(int p, int a, int b) const { return n + E * h + (p * h + a) * h + b; }
};

const double kInf = 1e300;

// One candidate shortest path between two distinct servers (reading R16):
// the ECMP shortest paths of a fat-tree.  id: 0 same edge; 1+a same pod;
// 1+h+a*h+b cross pod.  `fabric` = the non-access links of the path.
struct Path {
  int id;
  std::vector<int> fabric;
};

std::vector<Path> candidate_paths(const DC& dc, int u, int v) {
  std::vector<Path> out;
  int eu = dc.edge_of(u), ev = dc.edge_of(v);
  int pu = dc.pod_of_edge(eu), pv = dc.pod_of_edge(ev);
  if (eu == ev) {
    out.push_back(Path{0, {}});
  } else if (pu == pv) {
    for (int a = 0; a < dc.h; ++a) out.push_back(Path{1 + a, {dc.ea(eu, a), dc.ea(ev, a)}});
  } else {
    for (int a = 0; a < dc.h; ++a)
      for (int b = 0; b < dc.h; ++b)
        out.push_back(Path{1 + dc.h + a * dc.h + b,
                           {dc.ea(eu, a), dc.ac(pu, a, b), dc.ac(pv, a, b), dc.ea(ev, a)}});
  }
  return out;
}

double fabric_bottleneck(const DC& dc, const Path& p) {
  double b = kInf;
  for (int l : p.fabric) b = std::min(b, (double)dc.link[l]);
  return b;
}

// "shortest path that has the maximum available bandwidth": among the
// ECMP shortest paths pick the largest fabric bottleneck, first in (a, b)
// order on ties (reading R16).
Path widest_path(const DC& dc, int u, int v) {
  std::vector<Path> cands = candidate_paths(dc, u, v);
  size_t best = 0;
  double bb = fabric_bottleneck(dc, cands[0]);
  for (size_t i = 1; i < cands.size(); ++i) {
    double b = fabric_bottleneck(dc, cands[i]);
    if (b > bb) { bb = b; best = i; }
  }
  return cands[best];
}

// Widest fabric bottleneck from edge switch e to the edge switch of server v
// (SURVEY §8(a) a2): computed by enumerating the same candidate paths as
// widest_path for a representative server under e.
double fabric_widest_from_edge(const DC& dc, int e, int v) {
  int rep = e * dc.h;  // any server under e has the same fabric candidates
  if (dc.edge_of(v) == e) return kInf;
  std::vector<Path> cands = candidate_paths(dc, rep, v);
  double best = -1;
  for (const Path& p : cands) best = std::max(best, fabric_bottleneck(dc, p));
  return best;
}

// ---------------------------------------------------------------------------
// Options (DESIGN.md readings).
// ---------------------------------------------------------------------------
struct Opts {
  int method;       // 0 AHP, 1 TOPSIS, 2 BF (bin packing), 3 WF (spread): baselines of P:207-209
  double w[4];      // W over (CPU, RAM, Fragmentation, Bandwidth), T4 P:319-330 (R1)
  int ahp_rule;     // 0 literal (R8), 1 shifted
  int l1_mode;      // 0 pairwise comparison on W (R10), 1 L1 = W
  int path_filter;  // 1 filter on paths (R6), 0 paper-literal select-then-route
  int rank_once;    // 0 re-rank every pod step (R15); 1 rank once per request (R25)
  int bw_logical = 0;  // R2 alternative: the Bandwidth criterion is the logical bandwidth
};

// AHP pairwise cell for a scaled difference d (reading R8).
double ahp_cell(double d, int rule) {
  if (rule == 0) {
    if (d > 0) return d;
    if (d < 0) return 1.0 / (-d);
    return 1.0;
  }
  if (d > 0) return 1.0 + d;
  if (d < 0) return 1.0 / (1.0 - d);
  return 1.0;
}

// AHP local priority vector of m alternatives with values x:
// scale to [1,10] (R7) so that d_ij = 9 (x_i - x_j) / (hi - lo); pairwise
// matrix a_ij = cell(d_ij) (R8); normalise each column by its sum (R9,
// "both vectors are normalized"); priority = row mean (Eq. 10).
std::vector<double> ahp_priority(const std::vector<double>& x, int rule) {
  size_t m = x.size();
  std::vector<double> L(m, 0.0);
  if (m == 0) return L;
  double lo = *std::min_element(x.begin(), x.end());
  double hi = *std::max_element(x.begin(), x.end());
  if (hi == lo) {  // every value scales to 1: every cell is 1
    for (size_t i = 0; i < m; ++i) L[i] = 1.0 / (double)m;
    return L;
  }
  auto cell = [&](size_t i, size_t j) { return ahp_cell(9.0 * (x[i] - x[j]) / (hi - lo), rule); };
  // OpenMP over columns, then over rows (SURVEY §8(c) "OpenMP only across independent
  // requests or AHP rows"): every sum still runs sequentially in index order.
  std::vector<double> colsum(m, 0.0);
#pragma omp parallel for schedule(static) if (m >= 2048)
  for (long j = 0; j < (long)m; ++j)
    for (size_t i = 0; i < m; ++i) colsum[j] += cell(i, j);
#pragma omp parallel for schedule(static) if (m >= 2048)
  for (long i = 0; i < (long)m; ++i) {
    double s = 0.0;
    for (size_t j = 0; j < m; ++j) s += cell(i, j) / colsum[j];
    L[i] = s / (double)m;
  }
  return L;
}

// Criteria-level priority L1 (Eq. 9; reading R10).
void ahp_l1(const Opts& o, double L1[4]) {
  if (o.l1_mode == 1) {
    for (int c = 0; c < 4; ++c) L1[c] = o.w[c];
    return;
  }
  std::vector<double> w(o.w, o.w + 4);
  std::vector<double> l = ahp_priority(w, o.ahp_rule);
  for (int c = 0; c < 4; ++c) L1[c] = l[c];
}

struct Flow { int v; long D; };

struct RankOut {
  std::vector<uint8_t> mask;
  std::vector<double> score;
  int best = -1;
  std::vector<uint8_t> tie;  // R14 tie set at relative tolerance 1e-9
  long n_feasible = 0;
};

// One pod step's ranking (SURVEY §8(c) oracle steps 2.2-2.5).
RankOut rank(const DC& dc, const Opts& o, long dem_cpu, long dem_ram,
             const std::vector<Flow>& flows, const std::vector<int>& excluded) {
  RankOut r;
  r.mask.assign(dc.n, 0);
  r.score.assign(dc.n, 0.0);
  r.tie.assign(dc.n, 0);

  // a2: widest fabric bottleneck from every edge switch to every flow's server.
  std::vector<std::vector<double>> Fv(flows.size(), std::vector<double>(dc.E, 0.0));
  // Each table entry is independent: OpenMP over the edge switches (the per-entry
  // arithmetic is unchanged, so the table is identical at any thread count).
  if (o.path_filter)
    for (size_t f = 0; f < flows.size(); ++f) {
#pragma omp parallel for schedule(static) if (dc.E >= 512)
      for (int e = 0; e < dc.E; ++e) Fv[f][e] = fabric_widest_from_edge(dc, e, flows[f].v);
    }

  // a3: feasibility filter, Eq. 4-7, reading R6.
  for (int u = 0; u < dc.n; ++u) {
    bool ok = dc.cpu[u] >= dem_cpu && dc.ram[u] >= dem_ram;
    for (int x : excluded) if (x == u) ok = false;
    if (o.path_filter) {
      long sum_other = 0;
      for (const Flow& fl : flows) if (fl.v != u) sum_other += fl.D;
      if (dc.link[dc.access(u)] < sum_other) ok = false;
      for (size_t f = 0; f < flows.size(); ++f) {
        if (flows[f].v == u) continue;  // same server: host bus, no network
        if (dc.link[dc.access(flows[f].v)] < flows[f].D) ok = false;
        if (Fv[f][dc.edge_of(u)] < (double)flows[f].D) ok = false;
      }
    }
    r.mask[u] = ok ? 1 : 0;
  }
  std::vector<int> F;
  for (int u = 0; u < dc.n; ++u) if (r.mask[u]) F.push_back(u);
  r.n_feasible = (long)F.size();
  if (F.empty()) return r;

  // Criteria vector c^s_u U {f_u, bw^s_u} (readings R1-R3):
  // residual CPU, residual RAM, active flag, residual of u's access link.
  // R2's alternative reading (`bw_criterion = logical`): bw^s_u = "the sum of all bandwidth
  // capacity bw^s_uv with source on u", bw^s_uv (T1 P:90) read as the bottleneck of
  // the widest shortest path u-v (R16): min(access u, access v, widest fabric).
  std::vector<double> logical;
  if (o.bw_logical) {
    logical.assign(dc.n, 0.0);
    for (int u = 0; u < dc.n; ++u)
      for (int v = 0; v < dc.n; ++v) {
        if (v == u) continue;
        double b = std::min((double)dc.link[dc.access(u)], (double)dc.link[dc.access(v)]);
        b = std::min(b, fabric_bottleneck(dc, widest_path(dc, u, v)));
        logical[u] += b;
      }
  }
  auto crit = [&](int u, int c) -> double {
    switch (c) {
      case 0: return (double)dc.cpu[u];
      case 1: return (double)dc.ram[u];
      case 2: return (double)dc.active[u];
      default: return o.bw_logical ? logical[u] : (double)dc.link[dc.access(u)];
    }
  };

  if (o.method >= 2) {
    // BF / WF baselines ("the native algorithms offered by containers
    // orchestrators, BF (binpacking) and WF (spread)"; reading R27): the server's load is
    // the mean residual fraction of CPU and RAM, (cpu/cpu_cap + ram/ram_cap) / 2,
    // compared exactly as the integer cpu*ram_cap + ram*cpu_cap.  BF takes the most loaded
    // feasible server (smallest residual), WF the least loaded; ties lowest index.
    for (int u : F) {
      double key = (double)dc.cpu[u] * (double)dc.ram_cap + (double)dc.ram[u] * (double)dc.cpu_cap;
      r.score[u] = o.method == 2 ? -key : key;
    }
    int best = F[0];
    for (int u : F) if (r.score[u] > r.score[best]) best = u;
    r.best = best;
    for (int u : F) r.tie[u] = r.score[u] == r.score[best];  // integer keys: exact ties only
    return r;
  }
  if (o.method == 1) {
    // TOPSIS (readings R12-R13) over the feasible set F (R4).
    double N[4];
    for (int c = 0; c < 4; ++c) {
      double s = 0.0;
      for (int u : F) s += crit(u, c) * crit(u, c);
      N[c] = std::sqrt(s);
    }
    // evaluation vector M, normalised then weighted
    std::vector<std::vector<double>> V(F.size(), std::vector<double>(4, 0.0));
    for (size_t i = 0; i < F.size(); ++i)
      for (int c = 0; c < 4; ++c) V[i][c] = N[c] > 0 ? o.w[c] * crit(F[i], c) / N[c] : 0.0;
    double Ap[4], Am[4];
    for (int c = 0; c < 4; ++c) {
      Ap[c] = V[0][c];
      Am[c] = V[0][c];
      for (size_t i = 1; i < F.size(); ++i) {
        Ap[c] = std::max(Ap[c], V[i][c]);
        Am[c] = std::min(Am[c], V[i][c]);
      }
    }
    for (size_t i = 0; i < F.size(); ++i) {
      double dp = 0.0, dm = 0.0;
      for (int c = 0; c < 4; ++c) {
        dp += (V[i][c] - Ap[c]) * (V[i][c] - Ap[c]);
        dm += (V[i][c] - Am[c]) * (V[i][c] - Am[c]);
      }
      double Edp = std::sqrt(dp), Edm = std::sqrt(dm);
      r.score[F[i]] = (Edp + Edm) > 0 ? Edm / (Edp + Edm) : 0.0;
    }
  } else {
    // AHP (readings R7-R11): PG[u] = sum_c L1[c] * L2_c[u].
    double L1[4];
    ahp_l1(o, L1);
    for (int c = 0; c < 4; ++c) {
      std::vector<double> x(F.size());
      for (size_t i = 0; i < F.size(); ++i) x[i] = crit(F[i], c);
      std::vector<double> L2 = ahp_priority(x, o.ahp_rule);
      for (size_t i = 0; i < F.size(); ++i) r.score[F[i]] += L1[c] * L2[i];
    }
  }

  // a7: argmax, lowest index among exactly equal scores (R14).
  int best = F[0];
  for (int u : F) if (r.score[u] > r.score[best]) best = u;
  r.best = best;
  double smax = r.score[best];
  for (int u : F) if (r.score[u] >= smax - 1e-9 * std::fabs(smax)) r.tie[u] = 1;
  return r;
}

// ---------------------------------------------------------------------------
// Requests Req(N^c, E^c) in CSR form.
// ---------------------------------------------------------------------------
struct Req {
  int nC, nV;
  const int32_t *cpu_min, *cpu_max, *ram_min, *ram_max, *pod_of;
  const int32_t *src, *dst, *bw_min, *bw_max;
};

// Reading R24 / SPEC validate_request: returns the number of violations.
int validate(const Req& q, int P_limit_unused = 0) {
  (void)P_limit_unused;
  int bad = 0;
  if (q.nC <= 0) return 1;
  int maxp = -1;
  for (int i = 0; i < q.nC; ++i) {
    if (q.cpu_min[i] <= 0 || q.ram_min[i] <= 0) ++bad;
    if (q.cpu_min[i] > q.cpu_max[i] || q.ram_min[i] > q.ram_max[i]) ++bad;
    if (q.pod_of[i] < 0 || q.pod_of[i] >= q.nC) { ++bad; continue; }
    maxp = std::max(maxp, q.pod_of[i]);
  }
  std::vector<int> used(q.nC, 0);
  for (int i = 0; i < q.nC; ++i) if (q.pod_of[i] >= 0 && q.pod_of[i] < q.nC) used[q.pod_of[i]] = 1;
  for (int p = 0; p <= maxp; ++p) if (!used[p]) ++bad;
  for (int e = 0; e < q.nV; ++e) {
    if (q.src[e] < 0 || q.src[e] >= q.nC || q.dst[e] < 0 || q.dst[e] >= q.nC) { ++bad; continue; }
    if (q.src[e] == q.dst[e]) ++bad;
    if (q.bw_min[e] <= 0 || q.bw_min[e] > q.bw_max[e]) ++bad;
  }
  return bad;
}

struct Placement {
  int status = 0;
  std::vector<int> server, cpu_a, ram_a, bw_a, path;
};

struct Counters {
  long pod_steps = 0, retries = 0, excused_ties = 0, hint_mismatch = 0, servers_ranked = 0;
};

// One request against state `dc` (SURVEY §8(c) oracle algorithm).  On accept
// the state holds the placement; on reject it is restored (R20).  `hint`
// (nullable): per-container servers chosen by another implementation; at each
// pod step a hinted server inside the R14 tie set is adopted (lock-step resync).
Placement schedule_one(DC& dc, const Opts& o, const Req& q, const int32_t* hint, Counters& cnt) {
  Placement pl;
  pl.server.assign(q.nC, -1);
  pl.cpu_a.assign(q.nC, 0);
  pl.ram_a.assign(q.nC, 0);
  pl.bw_a.assign(q.nV, 0);
  pl.path.assign(q.nV, -1);
  if (validate(q) != 0) { pl.status = -1; return pl; }

  int P = 0;
  for (int i = 0; i < q.nC; ++i) P = std::max(P, q.pod_of[i] + 1);
  std::vector<long> pcpu(P, 0), pram(P, 0);
  for (int i = 0; i < q.nC; ++i) { pcpu[q.pod_of[i]] += q.cpu_min[i]; pram[q.pod_of[i]] += q.ram_min[i]; }
  std::vector<int> hint_pod(P, -1);
  if (hint)
    for (int i = q.nC - 1; i >= 0; --i) hint_pod[q.pod_of[i]] = hint[i];

  DC saved = dc;  // for the atomic rollback of a rejected request (R20)
  std::vector<int> srv(P, -1);
  std::vector<int> vpath(q.nV, -1);
  // R25 (rank once, "the resulting array is sorted on decreasing
  // order"): the ranking of the request's first pod step (pod 0, no flows, the
  // state at request start) orders the servers once; every pod step takes the first
  // server of that order that its own filter (R6, current residuals) admits.
  RankOut r0;
  if (o.rank_once) r0 = rank(dc, o, pcpu[0], pram[0], std::vector<Flow>(), std::vector<int>());

  for (int p = 0; p < P; ++p) {  // pods in ascending id (R15)
    std::vector<int> excluded;
    for (;;) {
      // Flows (R17): all vlinks between p and placed pods on server v form one flow D_v.
      std::map<int, long> agg;
      for (int e = 0; e < q.nV; ++e) {
        int pa = q.pod_of[q.src[e]], pb = q.pod_of[q.dst[e]];
        int other = -1;
        if (pa == p && pb != p && srv[pb] >= 0) other = pb;
        if (pb == p && pa != p && srv[pa] >= 0) other = pa;
        if (other >= 0) agg[srv[other]] += q.bw_min[e];
      }
      std::vector<Flow> flows;
      for (auto& kv : agg) flows.push_back(Flow{kv.first, kv.second});

      RankOut r = rank(dc, o, pcpu[p], pram[p], flows, excluded);
      cnt.pod_steps += 1;
      cnt.servers_ranked += dc.n;
      if (o.rank_once) {  // walk the request's order: best pod-0 score among the admitted servers
        int b = -1;
        for (int u = 0; u < dc.n; ++u)
          if (r.mask[u] && r0.mask[u] && (b < 0 || r0.score[u] > r0.score[b])) b = u;
        r.best = b;
        for (int u = 0; u < dc.n; ++u)
          r.tie[u] = b >= 0 && r.mask[u] && r0.mask[u] &&
                     r0.score[u] >= r0.score[b] - 1e-9 * std::fabs(r0.score[b]);
      }
      if (r.best < 0) {  // F empty: reject the whole request (R20)
        dc = saved;
        pl.status = 0;
        std::fill(pl.server.begin(), pl.server.end(), -1);
        std::fill(pl.cpu_a.begin(), pl.cpu_a.end(), 0);
        std::fill(pl.ram_a.begin(), pl.ram_a.end(), 0);
        std::fill(pl.bw_a.begin(), pl.bw_a.end(), 0);
        std::fill(pl.path.begin(), pl.path.end(), -1);
        return pl;
      }
      int u = r.best;
      int hp = hint_pod[p];
      // R14 resync on floating-point near-ties only: BF / WF decide on exact integer keys
      if (o.method < 2 && hp >= 0 && hp < dc.n && hp != u && r.tie[hp]) { u = hp; cnt.excused_ties += 1; }

      // a8 commit (Eq. 4-5; readings R16-R18).
      DC before = dc;
      dc.cpu[u] -= pcpu[p];
      dc.ram[u] -= pram[p];
      dc.active[u] = 1;
      bool failed = false;
      std::map<int, int> flow_path;
      for (const Flow& fl : flows) {  // ascending v
        if (fl.v == u) { flow_path[fl.v] = -1; continue; }
        Path path = widest_path(dc, u, fl.v);
        double bott = std::min({(double)dc.link[dc.access(u)], (double)dc.link[dc.access(fl.v)],
                                fabric_bottleneck(dc, path)});
        if (bott < (double)fl.D) { failed = true; break; }
        dc.link[dc.access(u)] -= fl.D;
        dc.link[dc.access(fl.v)] -= fl.D;
        for (int l : path.fabric) dc.link[l] -= fl.D;
        flow_path[fl.v] = path.id;
      }
      if (failed) {  // R18: exclude u*, undo this pod's commit, redo the pod step
        dc = before;
        excluded.push_back(u);
        cnt.retries += 1;
        continue;
      }
      // the hint names the server the other implementation finally committed the pod to: an
      // attempt that an R18 routing failure discards is no mismatch
      if (hp >= 0 && hp < dc.n && hp != u) cnt.hint_mismatch += 1;
      srv[p] = u;
      for (int e = 0; e < q.nV; ++e) {
        int pa = q.pod_of[q.src[e]], pb = q.pod_of[q.dst[e]];
        int other = -1;
        if (pa == p && pb != p && srv[pb] >= 0 && pb < p) other = pb;
        if (pb == p && pa != p && srv[pa] >= 0 && pa < p) other = pa;
        if (other >= 0) vpath[e] = flow_path[srv[other]];
      }
      break;
    }
  }

  // a9 request end: top-up (R19) in container index order, then vlink order.
  for (int i = 0; i < q.nC; ++i) {
    int u = srv[q.pod_of[i]];
    pl.server[i] = u;
    long extra_c = std::min<long>(q.cpu_max[i] - q.cpu_min[i], dc.cpu[u]);
    long extra_r = std::min<long>(q.ram_max[i] - q.ram_min[i], dc.ram[u]);
    dc.cpu[u] -= extra_c;
    dc.ram[u] -= extra_r;
    pl.cpu_a[i] = (int)(q.cpu_min[i] + extra_c);
    pl.ram_a[i] = (int)(q.ram_min[i] + extra_r);
  }
  for (int e = 0; e < q.nV; ++e) {
    int us = pl.server[q.src[e]], ud = pl.server[q.dst[e]];
    if (us == ud) {  // host bus carries intra-server traffic
      pl.bw_a[e] = q.bw_max[e];
      pl.path[e] = -1;
      continue;
    }
    // the vlink's path is the one its flow was routed on
    std::vector<Path> cands = candidate_paths(dc, us, ud);
    const Path* pp = nullptr;
    for (const Path& c : cands) if (c.id == vpath[e]) pp = &c;
    long resid = std::min(dc.link[dc.access(us)], dc.link[dc.access(ud)]);
    for (int l : pp->fabric) resid = std::min(resid, dc.link[l]);
    long extra = std::min<long>(q.bw_max[e] - q.bw_min[e], resid);
    dc.link[dc.access(us)] -= extra;
    dc.link[dc.access(ud)] -= extra;
    for (int l : pp->fabric) dc.link[l] -= extra;
    pl.bw_a[e] = (int)(q.bw_min[e] + extra);
    pl.path[e] = vpath[e];
  }
  pl.status = 1;
  return pl;
}

DC make_dc(int k, int cpu_cap, int ram_cap, int link_cap, const int32_t* cpu, const int32_t* ram,
           const uint8_t* active, const int32_t* link) {
  DC dc;
  dc.k = k;
  dc.h = k / 2;
  dc.n = k * k * k / 4;
  dc.E = k * k / 2;
  dc.L = 3 * k * k * k / 4;
  dc.cpu_cap = cpu_cap;
  dc.ram_cap = ram_cap;
  dc.link_cap = link_cap;
  dc.cpu.resize(dc.n);
  dc.ram.resize(dc.n);
  dc.active.resize(dc.n);
  dc.link.resize(dc.L);
  for (int u = 0; u < dc.n; ++u) {
    dc.cpu[u] = cpu ? cpu[u] : cpu_cap;
    dc.ram[u] = ram ? ram[u] : ram_cap;
    dc.active[u] = active ? active[u] : (dc.cpu[u] < cpu_cap || dc.ram[u] < ram_cap);
  }
  for (int l = 0; l < dc.L; ++l) dc.link[l] = link ? link[l] : link_cap;
  return dc;
}

Opts make_opts(int method, const double* w, int ahp_rule, int l1_mode, int path_filter, int rank_once = 0) {
  Opts o;
  o.rank_once = rank_once;
  o.method = method;
  for (int c = 0; c < 4; ++c) o.w[c] = w[c];
  o.ahp_rule = ahp_rule;
  o.l1_mode = l1_mode;
  // BF and WF "natively ignore the network requirements"; "a shortest-path search after the
  // allocation of servers": the CPU/RAM-only filter, then routing (R6 flag 0)
  o.path_filter = method >= 2 ? 0 : path_filter;
  return o;
}

}  // namespace

extern "C" {

// Rank one pod step (no state change).  score_out: double[n]; tie_out: R14 tie set.
int orc_rank(int k, int cpu_cap, int ram_cap, int link_cap, const int32_t* cpu, const int32_t* ram,
             const uint8_t* active, const int32_t* link, int method, const double* w, int ahp_rule,
             int l1_mode, int path_filter, int dem_cpu, int dem_ram, int nflow, const int32_t* flow_v,
             const int32_t* flow_D, int nexcl, const int32_t* excl, uint8_t* mask_out, double* score_out,
             int32_t* best_out, uint8_t* tie_out, int bw_logical) {
  DC dc = make_dc(k, cpu_cap, ram_cap, link_cap, cpu, ram, active, link);
  Opts o = make_opts(method, w, ahp_rule, l1_mode, path_filter);
  o.bw_logical = bw_logical;
  std::vector<Flow> flows;
  for (int f = 0; f < nflow; ++f) flows.push_back(Flow{flow_v[f], (long)flow_D[f]});
  std::sort(flows.begin(), flows.end(), [](const Flow& a, const Flow& b) { return a.v < b.v; });
  std::vector<int> ex(excl, excl + nexcl);
  RankOut r = rank(dc, o, dem_cpu, dem_ram, flows, ex);
  for (int u = 0; u < dc.n; ++u) {
    if (mask_out) mask_out[u] = r.mask[u];
    if (score_out) score_out[u] = r.score[u];
    if (tie_out) tie_out[u] = r.tie[u];
  }
  *best_out = r.best;
  return (int)r.n_feasible;
}

// AHP local priority of m values (exposed for pins).
void orc_ahp_priority(int m, const double* x, int rule, double* out) {
  std::vector<double> v(x, x + m);
  std::vector<double> L = ahp_priority(v, rule);
  for (int i = 0; i < m; ++i) out[i] = L[i];
}

void orc_ahp_l1(const double* w, int ahp_rule, int l1_mode, double* out) {
  Opts o = make_opts(0, w, ahp_rule, l1_mode, 1);
  ahp_l1(o, out);
}

// Widest ECMP shortest path between servers u != v on the given links.
// Returns path id; *fabric_out = its fabric bottleneck (1e300 if none).
int orc_widest_path(int k, const int32_t* link, int u, int v, double* fabric_out, int32_t* links_out,
                    int* nlinks_out) {
  DC dc = make_dc(k, 1, 1, 1, nullptr, nullptr, nullptr, link);
  Path p = widest_path(dc, u, v);
  *fabric_out = fabric_bottleneck(dc, p);
  *nlinks_out = (int)p.fabric.size();
  for (size_t i = 0; i < p.fabric.size(); ++i) links_out[i] = p.fabric[i];
  return p.id;
}

// Schedule a batch.  sequential=1: requests in order against the live state
// (arrays updated in place, P:206 online semantics); sequential=0: every
// request against the same input snapshot, nothing committed (R21), requests
// run in parallel over nthreads OpenMP threads.
// counters: [pod_steps, retries, excused_ties, hint_mismatch, servers_ranked].
int orc_schedule(int k, int cpu_cap, int ram_cap, int link_cap, int32_t* cpu, int32_t* ram, uint8_t* active,
                 int32_t* link, int method, const double* w, int ahp_rule, int l1_mode, int path_filter,
                 int rank_once, int sequential, int n_req, const int32_t* coff, const int32_t* cpu_min,
                 const int32_t* cpu_max, const int32_t* ram_min, const int32_t* ram_max,
                 const int32_t* pod_of, const int32_t* voff, const int32_t* vsrc, const int32_t* vdst,
                 const int32_t* bw_min, const int32_t* bw_max, const int32_t* hint, int32_t* status,
                 int32_t* server, int32_t* cpu_a, int32_t* ram_a, int32_t* bw_a, int32_t* path,
                 int64_t* counters, int nthreads) {
  DC base = make_dc(k, cpu_cap, ram_cap, link_cap, cpu, ram, active, link);
  Opts o = make_opts(method, w, ahp_rule, l1_mode, path_filter, rank_once);
  auto mkreq = [&](int r) {
    Req q;
    q.nC = coff[r + 1] - coff[r];
    q.nV = voff[r + 1] - voff[r];
    q.cpu_min = cpu_min + coff[r];
    q.cpu_max = cpu_max + coff[r];
    q.ram_min = ram_min + coff[r];
    q.ram_max = ram_max + coff[r];
    q.pod_of = pod_of + coff[r];
    q.src = vsrc + voff[r];
    q.dst = vdst + voff[r];
    q.bw_min = bw_min + voff[r];
    q.bw_max = bw_max + voff[r];
    return q;
  };
  auto emit = [&](int r, const Placement& pl) {
    status[r] = pl.status;
    for (int i = 0; i < coff[r + 1] - coff[r]; ++i) {
      server[coff[r] + i] = pl.server[i];
      cpu_a[coff[r] + i] = pl.cpu_a[i];
      ram_a[coff[r] + i] = pl.ram_a[i];
    }
    for (int e = 0; e < voff[r + 1] - voff[r]; ++e) {
      bw_a[voff[r] + e] = pl.bw_a[e];
      path[voff[r] + e] = pl.path[e];
    }
  };
  Counters total;
  if (sequential) {
    for (int r = 0; r < n_req; ++r) {
      Req q = mkreq(r);
      Placement pl = schedule_one(base, o, q, hint ? hint + coff[r] : nullptr, total);
      emit(r, pl);
    }
    for (int u = 0; u < base.n; ++u) {
      cpu[u] = (int32_t)base.cpu[u];
      ram[u] = (int32_t)base.ram[u];
      active[u] = (uint8_t)base.active[u];
    }
    for (int l = 0; l < base.L; ++l) link[l] = (int32_t)base.link[l];
  } else {
    std::vector<Counters> per(n_req);
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads > 0 ? nthreads : 1)
    for (int r = 0; r < n_req; ++r) {
      DC dc = base;  // private copy of the snapshot (R21)
      Req q = mkreq(r);
      Placement pl = schedule_one(dc, o, q, hint ? hint + coff[r] : nullptr, per[r]);
      emit(r, pl);
    }
    for (const Counters& c : per) {
      total.pod_steps += c.pod_steps;
      total.retries += c.retries;
      total.excused_ties += c.excused_ties;
      total.hint_mismatch += c.hint_mismatch;
      total.servers_ranked += c.servers_ranked;
    }
  }
  counters[0] = total.pod_steps;
  counters[1] = total.retries;
  counters[2] = total.excused_ties;
  counters[3] = total.hint_mismatch;
  counters[4] = total.servers_ranked;
  return 0;
}

}  // extern "C"


// ===========================================================================
// Departures and the discrete-event simulator (P:206 and P:391
// "a discrete event simulator"; P:396-398 the E2 campaign; T5 P:416-426 its metrics).
// ===========================================================================
namespace {

// Release an accepted placement: the exact inverse of its commit and top-up.
// f_u is re-derived as "some residual below capacity" (R22), so on a DC whose activity
// flags follow R22 apply-then-release is the identity.
void release_one(DC& dc, const Req& q, const Placement& pl) {
  for (int i = 0; i < q.nC; ++i) {
    int u = pl.server[i];
    dc.cpu[u] += pl.cpu_a[i];
    dc.ram[u] += pl.ram_a[i];
  }
  for (int e = 0; e < q.nV; ++e) {
    int us = pl.server[q.src[e]], ud = pl.server[q.dst[e]];
    if (us == ud) continue;  // host bus: no link carried it
    std::vector<Path> cands = candidate_paths(dc, us, ud);
    for (const Path& c : cands)
      if (c.id == pl.path[e]) {
        dc.link[dc.access(us)] += pl.bw_a[e];
        dc.link[dc.access(ud)] += pl.bw_a[e];
        for (int l : c.fabric) dc.link[l] += pl.bw_a[e];
      }
  }
  for (int i = 0; i < q.nC; ++i) {
    int u = pl.server[i];
    dc.active[u] = (dc.cpu[u] < dc.cpu_cap || dc.ram[u] < dc.ram_cap) ? 1 : 0;
  }
}

}  // namespace

extern "C" {

// Release the accepted requests (status 1) of a batch against the state, in request order.
void orc_release(int k, int cpu_cap, int ram_cap, int link_cap, int32_t* cpu, int32_t* ram, uint8_t* active,
                 int32_t* link, int n_req, const int32_t* coff, const int32_t* cpu_min, const int32_t* cpu_max,
                 const int32_t* ram_min, const int32_t* ram_max, const int32_t* pod_of, const int32_t* voff,
                 const int32_t* vsrc, const int32_t* vdst, const int32_t* bw_min, const int32_t* bw_max,
                 const int32_t* status, const int32_t* server, const int32_t* cpu_a, const int32_t* ram_a,
                 const int32_t* bw_a, const int32_t* path) {
  DC dc = make_dc(k, cpu_cap, ram_cap, link_cap, cpu, ram, active, link);
  for (int r = 0; r < n_req; ++r) {
    if (status[r] != 1) continue;
    Req q{coff[r + 1] - coff[r], voff[r + 1] - voff[r], cpu_min + coff[r], cpu_max + coff[r], ram_min + coff[r],
          ram_max + coff[r], pod_of + coff[r], vsrc + voff[r], vdst + voff[r], bw_min + voff[r], bw_max + voff[r]};
    Placement pl;
    pl.server.assign(server + coff[r], server + coff[r + 1]);
    pl.cpu_a.assign(cpu_a + coff[r], cpu_a + coff[r + 1]);
    pl.ram_a.assign(ram_a + coff[r], ram_a + coff[r + 1]);
    pl.bw_a.assign(bw_a + voff[r], bw_a + voff[r + 1]);
    pl.path.assign(path + voff[r], path + voff[r + 1]);
    release_one(dc, q, pl);
  }
  for (int u = 0; u < dc.n; ++u) {
    cpu[u] = (int32_t)dc.cpu[u];
    ram[u] = (int32_t)dc.ram[u];
    active[u] = (uint8_t)dc.active[u];
  }
  for (int l = 0; l < dc.L; ++l) link[l] = (int32_t)dc.link[l];
}

// Discrete-event simulation (reading R28; SPEC S:519 event loop).  Ticks
// t = 0, 1, 2, ...: (1) release the requests whose start + duration == t; (2) enqueue the
// requests arriving at t (ascending id); (3) offer queued requests in FIFO order to the
// scheduler on the live state (sequential semantics): an accepted request leaves
// the queue and holds its resources for `duration` ticks; a refused one stays queued
// (with hol = 1 the scan of this tick stops at it, head-of-line blocking).  The run ends
// after the first tick at which no request is queued or still to arrive ("events", T5
// "# Events"), or after max_ticks ticks (requests still queued are then rejected).
// Per request: start tick (-1 never), attempts, and its final placement; per tick:
// active servers |N^s'|, active links |E^s'| (residual below capacity) and
// the queue length after the tick.  totals: [events, attempts, accepted, pod_steps,
// retries, excused_ties, hint_mismatch].
void orc_simulate(int k, int cpu_cap, int ram_cap, int link_cap, int32_t* cpu, int32_t* ram, uint8_t* active,
                  int32_t* link, int method, const double* w, int ahp_rule, int l1_mode, int path_filter,
                  int n_req, const int32_t* coff, const int32_t* cpu_min, const int32_t* cpu_max,
                  const int32_t* ram_min, const int32_t* ram_max, const int32_t* pod_of, const int32_t* voff,
                  const int32_t* vsrc, const int32_t* vdst, const int32_t* bw_min, const int32_t* bw_max,
                  const int32_t* arrival, const int32_t* duration, int max_ticks, int hol, const int32_t* hint,
                  int32_t* start, int32_t* attempts, int32_t* status, int32_t* server, int32_t* cpu_a,
                  int32_t* ram_a, int32_t* bw_a, int32_t* path, int32_t* tick_servers, int32_t* tick_links,
                  int32_t* tick_queue, int64_t* totals) {
  DC dc = make_dc(k, cpu_cap, ram_cap, link_cap, cpu, ram, active, link);
  Opts o = make_opts(method, w, ahp_rule, l1_mode, path_filter);
  auto mkreq = [&](int r) {
    return Req{coff[r + 1] - coff[r], voff[r + 1] - voff[r], cpu_min + coff[r], cpu_max + coff[r], ram_min + coff[r],
               ram_max + coff[r], pod_of + coff[r], vsrc + voff[r], vdst + voff[r], bw_min + voff[r], bw_max + voff[r]};
  };
  std::vector<Placement> placed(n_req);
  std::vector<int> order(n_req);
  for (int r = 0; r < n_req; ++r) {
    order[r] = r;
    start[r] = -1;
    attempts[r] = 0;
    status[r] = 0;
  }
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return arrival[a] < arrival[b]; });
  std::vector<int> queue;
  Counters cnt;
  long n_attempts = 0, accepted = 0;
  size_t next_arrival = 0;
  int t = 0;
  for (; t < max_ticks; ++t) {
    // (1) departures first
    for (int r = 0; r < n_req; ++r)
      if (start[r] >= 0 && start[r] + duration[r] == t) release_one(dc, mkreq(r), placed[r]);
    // (2) arrivals
    while (next_arrival < order.size() && arrival[order[next_arrival]] == t) queue.push_back(order[next_arrival++]);
    // (3) FIFO scan of the queue
    std::vector<int> left;
    bool blocked = false;
    for (int r : queue) {
      if (blocked) { left.push_back(r); continue; }
      Req q = mkreq(r);
      Placement pl = schedule_one(dc, o, q, hint ? hint + coff[r] : nullptr, cnt);
      ++n_attempts;
      ++attempts[r];
      if (pl.status == 1) {
        placed[r] = pl;
        start[r] = t;
        status[r] = 1;
        ++accepted;
      } else {
        if (pl.status == -1) status[r] = -1;
        if (pl.status == -1) continue;  // invalid: dropped from the queue
        left.push_back(r);
        if (hol) blocked = true;
      }
    }
    queue.swap(left);
    int as = 0, al = 0;
    for (int u = 0; u < dc.n; ++u) as += dc.active[u] ? 1 : 0;
    for (int l = 0; l < dc.L; ++l) al += dc.link[l] < dc.link_cap ? 1 : 0;
    tick_servers[t] = as;
    tick_links[t] = al;
    tick_queue[t] = (int)queue.size();
    if (queue.empty() && next_arrival == order.size()) { ++t; break; }
  }
  for (int r = 0; r < n_req; ++r) {
    const Placement& pl = placed[r];
    for (int i = 0; i < coff[r + 1] - coff[r]; ++i) {
      server[coff[r] + i] = status[r] == 1 ? pl.server[i] : -1;
      cpu_a[coff[r] + i] = status[r] == 1 ? pl.cpu_a[i] : 0;
      ram_a[coff[r] + i] = status[r] == 1 ? pl.ram_a[i] : 0;
    }
    for (int e = 0; e < voff[r + 1] - voff[r]; ++e) {
      bw_a[voff[r] + e] = status[r] == 1 ? pl.bw_a[e] : 0;
      path[voff[r] + e] = status[r] == 1 ? pl.path[e] : -1;
    }
  }
  for (int u = 0; u < dc.n; ++u) {
    cpu[u] = (int32_t)dc.cpu[u];
    ram[u] = (int32_t)dc.ram[u];
    active[u] = (uint8_t)dc.active[u];
  }
  for (int l = 0; l < dc.L; ++l) link[l] = (int32_t)dc.link[l];
  totals[0] = t;
  totals[1] = n_attempts;
  totals[2] = accepted;
  totals[3] = cnt.pod_steps;
  totals[4] = cnt.retries;
  totals[5] = cnt.excused_ties;
  totals[6] = cnt.hint_mismatch;
}

}  // extern "C"

// ===========================================================================
// General topology: the "modified Dijkstra" of P:383-386
// (§V-D) on an arbitrary undirected graph G^s(N^s, E^s) (§II-A), not
// only the fat-tree closed form above.  "A modified Dijkstra algorithm is used
// to compute the shortest path that has the maximum available bandwidth
// between the hosting servers"; links are undirected and u->v equals
// v->u.  Reading R26: a link is usable for a flow of
// demand D iff its residual >= D; among the usable paths the path has the
// fewest hops, then the largest bottleneck (min residual over its links), then
// the lexicographically smallest vertex sequence.
// ===========================================================================
namespace {

struct Graph {
  int V = 0;
  std::vector<std::vector<std::pair<int, long>>> adj;  // (neighbour, residual), both directions
};

Graph make_graph(int V, int nl, const int32_t* lu, const int32_t* lv, const int32_t* lr) {
  Graph G;
  G.V = V;
  G.adj.assign(V, {});
  for (int l = 0; l < nl; ++l) {
    G.adj[lu[l]].push_back({lv[l], (long)lr[l]});
    G.adj[lv[l]].push_back({lu[l], (long)lr[l]});
  }
  return G;
}

// Label of a vertex = the best (hops, width) over usable paths from the vertex to
// the root; better = fewer hops, then wider.  The order is isotone (extending two
// paths by the same link keeps their order), so Dijkstra's label-setting is exact.
struct Label {
  long hops;     // -1 = unreached
  double width;  // bottleneck; the root has +inf
};

bool better(long h1, double w1, long h2, double w2) { return h1 < h2 || (h1 == h2 && w1 > w2); }

// Modified Dijkstra from `root` over the links with residual >= demand.
std::vector<Label> dijkstra(const Graph& G, int root, long demand) {
  std::vector<Label> lab(G.V, Label{-1, 0.0});
  std::vector<char> done(G.V, 0);
  // priority queue ordered by label (a plain O(V^2) selection: slow and obviously right)
  lab[root] = Label{0, kInf};
  for (;;) {
    int v = -1;
    for (int x = 0; x < G.V; ++x)
      if (!done[x] && lab[x].hops >= 0 &&
          (v < 0 || better(lab[x].hops, lab[x].width, lab[v].hops, lab[v].width)))
        v = x;
    if (v < 0) break;
    done[v] = 1;
    for (const auto& e : G.adj[v]) {
      if (e.second < demand) continue;  // link not usable for this demand (R26)
      long h = lab[v].hops + 1;
      double w = std::min(lab[v].width, (double)e.second);
      Label& t = lab[e.first];
      if (!done[e.first] && (t.hops < 0 || better(h, w, t.hops, t.width))) t = Label{h, w};
    }
  }
  return lab;
}

// One (src, dst, demand) query: labels from dst, then the walk from src that takes, at
// every vertex, the smallest-id neighbour through which an optimal path continues
// (one hop closer to dst, bottleneck still >= the optimum): the lexicographically
// smallest vertex sequence among the optimal paths.  Returns hops (-1 if no usable path).
long widest_shortest(const Graph& G, int src, int dst, long demand, double* bottleneck, std::vector<int>* path) {
  std::vector<Label> lab = dijkstra(G, dst, demand);
  path->clear();
  if (lab[src].hops < 0) {
    *bottleneck = -1;
    return -1;
  }
  const double B = lab[src].width;
  int v = src;
  path->push_back(v);
  while (v != dst) {
    int next = -1;
    for (const auto& e : G.adj[v]) {
      int w = e.first;
      if (e.second < demand || lab[w].hops != lab[v].hops - 1) continue;
      if (std::min((double)e.second, lab[w].width) < B) continue;
      if (next < 0 || w < next) next = w;
    }
    v = next;
    path->push_back(v);
  }
  *bottleneck = B;
  return lab[src].hops;
}

}  // namespace

extern "C" {

// Batch of widest-shortest path queries on one immutable graph (element-wise
// identical to sequential calls).  Vertices 0..V-1; link l joins lu[l] and lv[l] with
// residual lr[l].  Outputs per query q: bn[q] bottleneck (-1 infeasible), hops[q] (-1
// infeasible), path[q * (max_hops + 1) ...] the vertex sequence src..dst (-1 padded; all -1
// when infeasible or when the path has more than max_hops links).
void orc_graph_paths(int V, int nl, const int32_t* lu, const int32_t* lv, const int32_t* lr, int nq,
                     const int32_t* src, const int32_t* dst, const int32_t* demand, int32_t* bn, int32_t* hops,
                     int32_t* path, int max_hops, int nthreads) {
  Graph G = make_graph(V, nl, lu, lv, lr);
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads > 0 ? nthreads : 1)
  for (int q = 0; q < nq; ++q) {
    double b = 0;
    std::vector<int> p;
    long h = widest_shortest(G, src[q], dst[q], demand[q], &b, &p);
    bn[q] = (int32_t)b;
    hops[q] = (int32_t)h;
    if (path) {  // the row holds the whole path, or is all -1 (infeasible, or longer than max_hops)
      const bool fits = h >= 0 && h <= max_hops;
      for (int i = 0; i <= max_hops; ++i)
        path[(size_t)q * (max_hops + 1) + i] = (fits && i < (int)p.size()) ? p[i] : -1;
    }
  }
}

// Logical bandwidth criterion (reading R2, alternative `bw_criterion=logical`:
// "sum of all bandwidth capacity bw^s_uv with source on u"): for each server
// u < ns, the sum over servers v != u of the bottleneck of the widest shortest path
// u -> v with every link usable (demand 0); unreachable servers add 0.
void orc_logical_bandwidth(int V, int ns, int nl, const int32_t* lu, const int32_t* lv, const int32_t* lr,
                           int64_t* out, int nthreads) {
  Graph G = make_graph(V, nl, lu, lv, lr);
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads > 0 ? nthreads : 1)
  for (int u = 0; u < ns; ++u) {
    std::vector<Label> lab = dijkstra(G, u, 0);
    int64_t s = 0;
    for (int v = 0; v < ns; ++v)
      if (v != u && lab[v].hops >= 0) s += (int64_t)lab[v].width;
    out[u] = s;
  }
}

}  // extern "C"
