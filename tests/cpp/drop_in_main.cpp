// The reference's own criterion-7 loop (acceptance_main.cpp:367-416), run
// twice in lock step: once on kvsched::GlobalScheduler (the unmodified
// reference, compiled from its sources) and once on the drop-in
// kvsched::b200::GlobalScheduler (include/e2sched.hpp over the C ABI).
// Every Decision field and cost double must match.  Exit 0 on success.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <deque>

#include "e2sched.hpp"
#include "kvsched/workload.hpp"

using namespace kvsched;

static bool same(const Decision& a, const Decision& b) {
  if (a.branch != b.branch || a.gpu != b.gpu || a.redirected != b.redirected ||
      a.pre_redirect_gpu != b.pre_redirect_gpu || a.cached_len != b.cached_len || a.missed_len != b.missed_len ||
      a.missed_on_chosen != b.missed_on_chosen || a.costs.size() != b.costs.size() ||
      a.decode_ratios != b.decode_ratios)
    return false;
  for (size_t i = 0; i < a.costs.size(); ++i) {
    const CostBreakdown &x = a.costs[i].cost, &y = b.costs[i].cost;
    if (a.costs[i].gpu != b.costs[i].gpu || x.current_load_ms != y.current_load_ms ||
        x.eviction_ms != y.eviction_ms || x.prefill_ms != y.prefill_ms ||
        x.eviction_infeasible != y.eviction_infeasible)
      return false;
  }
  return true;
}

// snapshot(now) of both sides (global_scheduler.cpp:375-394); the
// reference's raw hit deques are read through the window like any of its
// reads (prefix_tree.cpp:37-43).
static bool same_snapshot(ClusterSnapshot a, const ClusterSnapshot& b, SimTime horizon) {
  if (a.now != b.now || a.n_gpus != b.n_gpus || a.redirects != b.redirects || a.nodes.size() != b.nodes.size() ||
      a.gpus.size() != b.gpus.size())
    return false;
  for (size_t i = 0; i < a.nodes.size(); ++i) {
    auto& x = a.nodes[i];
    const auto& y = b.nodes[i];
    for (auto it = x.hits.begin(); it != x.hits.end();) {
      auto& v = it->second;
      v.erase(v.begin(), std::find_if(v.begin(), v.end(), [&](SimTime t) { return !(t < a.now - horizon); }));
      it = v.empty() ? x.hits.erase(it) : std::next(it);
    }
    if (x.id != y.id || x.parent_id != y.parent_id || x.edge != y.edge || x.caching_gpus != y.caching_gpus ||
        x.hits != y.hits || x.last_access != y.last_access || x.pin_count != y.pin_count)
      return false;
  }
  for (size_t g = 0; g < a.gpus.size(); ++g) {
    const auto &x = a.gpus[g], &y = b.gpus[g];
    if (x.id != y.id || x.inflight_cached != y.inflight_cached || x.inflight_prompt != y.inflight_prompt ||
        x.scheduled.size() != y.scheduled.size() || x.completed.size() != y.completed.size())
      return false;
    for (size_t i = 0; i < x.scheduled.size(); ++i)
      if (x.scheduled[i].t != y.scheduled[i].t || x.scheduled[i].missed != y.scheduled[i].missed ||
          x.scheduled[i].est_output != y.scheduled[i].est_output)
        return false;
    for (size_t i = 0; i < x.completed.size(); ++i)
      if (x.completed[i].t != y.completed[i].t || x.completed[i].output != y.completed[i].output) return false;
  }
  return true;
}

template <typename S>
static void step(S& s, std::vector<std::deque<std::pair<const TokenSeq*, int64_t>>>& cached, const Request& r,
                 SimTime now, int64_t trunk, const Decision& d) {
  s.note_prefill_cached(r.prompt, d.gpu, now);
  cached[d.gpu].push_back({&r.prompt, static_cast<int64_t>(r.prompt.size()) - trunk});
  auto cached_tokens = [&](GpuId g) {
    if constexpr (std::is_same_v<S, kvsched::GlobalScheduler>)
      return s.mirror().cached_tokens(g);
    else
      return s.cached_tokens(g);
  };
  while (cached_tokens(d.gpu) > 150000 && !cached[d.gpu].empty()) {
    EvictedRange range;
    range.seq = *cached[d.gpu].front().first;
    range.tail_len = cached[d.gpu].front().second;
    cached[d.gpu].pop_front();
    s.note_eviction(range, d.gpu, now);
  }
}

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? std::atoll(argv[1]) : 3000;
  WorkloadSpec spec = WorkloadSpec::archetype_default(Archetype::Toolbench);
  spec.request_count = n;
  Corpus corpus = generate(spec, 13);
  assign_poisson_arrivals(corpus, 2000.0, 14);
  const std::vector<Request> reqs = to_requests(corpus);
  const int64_t trunk = spec.system_prompt_len + spec.branch_len;
  SchedulerConfig cfg;
  cfg.kv_capacity_tokens = 200000;
  cfg.history_window_ms = 10000.0;
  kvsched::GlobalScheduler ref(4, cfg, TimeModel{}, GlobalPolicy{});
  kvsched::b200::GlobalScheduler dut(4, cfg, TimeModel{}, GlobalPolicy{});
  std::vector<std::deque<std::pair<const TokenSeq*, int64_t>>> ca(4), cb(4);
  SimTime now = 0;
  double t_ref = 0, t_dut = 0;  // seconds spent in each side's calls
  using clk = std::chrono::steady_clock;
  for (size_t i = 0; i < reqs.size(); ++i) {
    const Request& r = reqs[i];
    now = std::max(now, r.arrival_ms);
    auto t0 = clk::now();
    const Decision a = ref.schedule_request(r, now);
    auto t1 = clk::now();
    const Decision b = dut.schedule_request(r, now);
    auto t2 = clk::now();
    t_ref += std::chrono::duration<double>(t1 - t0).count();
    t_dut += std::chrono::duration<double>(t2 - t1).count();
    if (!same(a, b)) {
      std::printf("MISMATCH at request %zu\n", i);
      return 1;
    }
    t0 = clk::now();
    step(ref, ca, r, now, trunk, a);
    if (i >= 2000) ref.note_finished(reqs[i - 2000].id, now, reqs[i - 2000].output_len);
    t1 = clk::now();
    step(dut, cb, r, now, trunk, b);
    if (i >= 2000) dut.note_finished(reqs[i - 2000].id, now, reqs[i - 2000].output_len);
    t2 = clk::now();
    t_ref += std::chrono::duration<double>(t1 - t0).count();
    t_dut += std::chrono::duration<double>(t2 - t1).count();
    if ((i + 1) % 1000 == 0 && !same_snapshot(ref.snapshot(now), dut.snapshot(now), cfg.history_window_ms)) {
      std::printf("snapshot MISMATCH after request %zu\n", i);
      return 1;
    }
  }
  const GlobalStats sa = ref.stats(), sb = dut.stats();
  if (sa.exploit != sb.exploit || sa.explore != sb.explore || sa.redirected != sb.redirected ||
      sa.rebalance_installs != sb.rebalance_installs || sa.tree_reads != sb.tree_reads) {
    std::printf("stats differ\n");
    return 1;
  }
  std::printf("drop-in OK: %lld decisions identical (%s backend)\n", (long long)n, e2_backend());
  std::printf("per-call loop: reference %.0f requests/s, %s %.0f requests/s\n", n / t_ref, e2_backend(), n / t_dut);
  return 0;
}
