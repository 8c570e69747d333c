// e2sched.hpp — drop-in C++ face of the C ABI for the reference's callers.
//
// kvsched::b200::GlobalScheduler has the member signatures of
// kvsched::GlobalScheduler (proj/include/kvsched/global_scheduler.hpp:99-161)
// and throws the same exception types, so a caller such as the simulator
// (simulator.cpp:62, 92, 139, 154, 214, 221) or the criterion-7 driver
// (acceptance_main.cpp:383-405) switches by changing the class name and
// linking libe2sched.so.  The reference's types come from its own headers.
//
// Not provided: mirror() (the tree lives in HBM; use cached_tokens(),
// debug_dump(), snapshot() or match() instead — a host PrefixTree
// materialisation would be an export, a slow path).  snapshot() is provided;
// its NodeSnapshot::hits hold the in-window stamps (t >= now - H), what
// every read of the reference sees after its lazy prune.
#pragma once

#include <map>
#include <string>
#include <vector>

#include "e2sched.h"
#include "kvsched/global_scheduler.hpp"

namespace kvsched {
namespace b200 {

class GlobalScheduler {
 public:
  GlobalScheduler(int n_gpus, const SchedulerConfig& config, const TimeModel& model, const GlobalPolicy& policy)
      : n_(n_gpus), config_(config), model_(model), policy_(policy) {
    e2_sched_cfg c{config.history_window_ms, config.th_bal,        config.imbal_ratio,
                   config.priority_groups,   config.kv_capacity_tokens, config.default_output_len};
    e2_time_model m{model.prefill_base_ms, model.prefill_per_token_ms, model.decode_per_token_ms,
                    model.iteration_base_ms};
    e2_policy p{policy.mode == GlobalMode::RoundRobin ? E2_MODE_ROUND_ROBIN : E2_MODE_PREFIX_AWARE,
                policy.rebalance ? 1 : 0, policy.autoscale ? 1 : 0, policy.pd_balance ? 1 : 0};
    check(e2_create(n_gpus, &c, &m, &p, &h_), nullptr);
    costs_.resize(n_gpus + 1);
    ratios_.resize(n_gpus);
  }
  ~GlobalScheduler() { e2_destroy(h_); }
  GlobalScheduler(const GlobalScheduler&) = delete;
  GlobalScheduler& operator=(const GlobalScheduler&) = delete;

  Decision schedule_request(const Request& req, SimTime now) {
    e2_decision d;
    check(e2_schedule(h_, req.prompt.data(), (int64_t)req.prompt.size(), req.id, req.arrival_ms, now, &d,
                      costs_.data(), ratios_.data()),
          h_);
    return convert(d);
  }
  Decision decide(const Request& req, SimTime now) {
    e2_decision d;
    check(e2_decide(h_, req.prompt.data(), (int64_t)req.prompt.size(), req.id, now, &d, costs_.data(),
                    ratios_.data()),
          h_);
    return convert(d);
  }

  void note_admitted(RequestId id, SimTime now) { check(e2_note_admitted(h_, id, now), h_); }
  void note_prefill_cached(const TokenSeq& prompt, GpuId gpu, SimTime now) {
    check(e2_note_prefill_cached(h_, prompt.data(), (int64_t)prompt.size(), gpu, now), h_);
  }
  void note_eviction(const EvictedRange& range, GpuId gpu, SimTime now) {
    check(e2_note_eviction(h_, range.seq.data(), (int64_t)range.seq.size(), range.tail_len, gpu, now), h_);
  }
  void note_finished(RequestId id, SimTime now, int64_t output_len) {
    check(e2_note_finished(h_, id, now, output_len), h_);
  }

  double decode_ratio(GpuId gpu) const {
    double v = 0;
    check(e2_decode_ratio(h_, gpu, &v), h_);
    return v;
  }
  double gpu_load_ms(GpuId gpu, SimTime now) {
    double v = 0;
    check(e2_gpu_load_ms(h_, gpu, now, &v), h_);
    return v;
  }
  int64_t prune_dead_nodes(SimTime now) {
    int64_t v = 0;
    check(e2_prune_dead_nodes(h_, now, &v), h_);
    return v;
  }
  // mirror().cached_tokens(gpu) — the read the criterion-7 driver makes
  int64_t cached_tokens(GpuId gpu) const {
    int64_t v = 0;
    check(e2_cached_tokens(h_, gpu, &v), h_);
    return v;
  }
  std::string debug_dump(SimTime now) const {
    size_t need = 0;
    check(e2_debug_dump(h_, now, nullptr, 0, &need), h_);
    std::string s(need + 1, '\0');
    check(e2_debug_dump(h_, now, s.data(), s.size(), &need), h_);
    s.resize(need);
    return s;
  }
  std::map<GpuId, GpuId> redirects() const {
    std::vector<int32_t> r(n_);
    check(e2_redirects(h_, r.data()), h_);
    std::map<GpuId, GpuId> m;
    for (int g = 0; g < n_; ++g)
      if (r[g] >= 0) m[g] = r[g];
    return m;
  }
  GlobalStats stats() const {
    e2_stats s;
    check(e2_get_stats(h_, &s), h_);
    GlobalStats o;
    o.exploit = s.exploit;
    o.explore = s.explore;
    o.decode_pressure = s.decode_pressure;
    o.round_robin = s.round_robin;
    o.redirected = s.redirected;
    o.rebalance_installs = s.rebalance_installs;
    o.autoscale_events = s.autoscale_events;
    o.tree_reads = s.tree_reads;
    return o;
  }
  // snapshot(now) — global_scheduler.cpp:375-394
  ClusterSnapshot snapshot(SimTime now) {
    ClusterSnapshot snap;
    snap.now = now;
    snap.n_gpus = n_;
    snap.config = config_;
    snap.model = model_;
    snap.policy = policy_;
    int64_t nn = 0, nt = 0, ns = 0;
    check(e2_export_size(h_, &nn, &nt), h_);
    std::vector<e2_node> nodes(nn);
    std::vector<int32_t> tok(nt);
    std::vector<double> la(nn * n_);
    std::vector<int64_t> hits(nn * n_);
    check(e2_export(h_, now, nodes.data(), tok.data(), la.data(), hits.data()), h_);
    check(e2_export_hit_stamps(h_, now, nullptr, 0, &ns), h_);
    std::vector<double> st(ns);
    check(e2_export_hit_stamps(h_, now, st.data(), ns, &ns), h_);
    int64_t k = 0;
    for (int64_t i = 0; i < nn; ++i) {
      PrefixTree::NodeSnapshot o;
      o.id = nodes[i].id;
      o.parent_id = nodes[i].parent_id;
      o.edge.assign(tok.begin() + nodes[i].edge_off, tok.begin() + nodes[i].edge_off + nodes[i].edge_len);
      for (int g = 0; g < n_; ++g) {
        if ((nodes[i].caching_mask >> g) & 1ull) o.caching_gpus.push_back(g);
        if ((nodes[i].last_access_mask >> g) & 1ull) o.last_access[g] = la[i * n_ + g];
        const int64_t c = hits[i * n_ + g];
        if (c > 0) o.hits[g].assign(st.begin() + k, st.begin() + k + c);
        k += c;
      }
      o.pin_count = (int)nodes[i].pin_count;
      snap.nodes.push_back(std::move(o));
    }
    for (int g = 0; g < n_; ++g) {
      ClusterSnapshot::GpuSnap gs;
      gs.id = g;
      int64_t nsch = 0, ncomp = 0;
      check(e2_window_sizes(h_, g, now, &nsch, &ncomp, &gs.inflight_cached, &gs.inflight_prompt), h_);
      std::vector<double> t(nsch), ct(ncomp);
      std::vector<int64_t> m(nsch), e(nsch), co(ncomp);
      check(e2_window_entries(h_, g, now, t.data(), m.data(), e.data(), ct.data(), co.data()), h_);
      for (int64_t i = 0; i < nsch; ++i) gs.scheduled.push_back({t[i], m[i], e[i]});
      for (int64_t i = 0; i < ncomp; ++i) gs.completed.push_back({ct[i], co[i]});
      snap.gpus.push_back(std::move(gs));
    }
    snap.redirects = redirects();
    return snap;
  }
  int n_gpus() const { return n_; }
  const SchedulerConfig& config() const { return config_; }
  const TimeModel& model() const { return model_; }
  e2_handle* handle() { return h_; }

 private:
  static void check(int rc, const e2_handle* h) {
    if (rc == E2_OK) return;
    const std::string msg = e2_last_error(h);
    switch (rc) {
      case E2_ERR_CONFIG: throw ConfigError(msg);
      case E2_ERR_NO_ADMISSIBLE: throw NoAdmissibleGpu(msg);
      case E2_ERR_SIM: throw SimError(msg);
      default: throw std::runtime_error("e2sched: " + msg);
    }
  }

  Decision convert(const e2_decision& d) const {
    Decision o;
    o.request = d.request;
    o.branch = d.branch == E2_BRANCH_EXPLOIT   ? Branch::Exploit
               : d.branch == E2_BRANCH_EXPLORE ? Branch::Explore
               : d.branch == E2_BRANCH_DECODE_PRESSURE ? Branch::ExploreDecodePressure
                                                       : Branch::RoundRobin;
    o.gpu = d.gpu;
    o.redirected = d.redirected != 0;
    o.pre_redirect_gpu = d.pre_redirect_gpu;
    o.cached_len = d.cached_len;
    o.missed_len = d.missed_len;
    o.missed_on_chosen = d.missed_on_chosen;
    for (int i = 0; i < d.n_costs; ++i) {
      GpuCandidateCost c;
      c.gpu = costs_[i].gpu;
      c.cost.current_load_ms = costs_[i].current_load_ms;
      c.cost.eviction_ms = costs_[i].eviction_ms;
      c.cost.prefill_ms = costs_[i].prefill_ms;
      c.cost.eviction_infeasible = costs_[i].eviction_infeasible != 0;
      o.costs.push_back(c);
    }
    if (d.has_ratios)
      for (int g = 0; g < n_; ++g) o.decode_ratios[g] = ratios_[g];
    return o;
  }

  int n_;
  SchedulerConfig config_;
  TimeModel model_;
  GlobalPolicy policy_;
  e2_handle* h_ = nullptr;
  std::vector<e2_cost> costs_;
  std::vector<double> ratios_;
};

}  // namespace b200
}  // namespace kvsched
