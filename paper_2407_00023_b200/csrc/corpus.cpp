// corpus.cpp — corpus / trace files and the corpus study.
//
// Host C++ around the hot path (input and study tooling, like the trace
// generator in workload_gen.cpp):
//   * corpus text files: one request per line, "id [arrival_ms] tok... out"
//     (workload.cpp:329-387 — the arrival is written with "%.3f" and
//     recognised by its decimal point);
//   * request-trace CSV files with a header row: arrival_s, prompt_len,
//     output_len, stably sorted by arrival (workload.cpp:389-437);
//   * synthesize_from_trace: toolbench-shaped content for a trace's lengths
//     (workload.cpp:439-484), the same RNG draw sequence;
//   * analyze: the corpus study of workload.cpp:513-601.
//
// The study is computed without building a radix tree.  With every prompt
// inserted into an infinite-capacity tree, the tree's nodes are exactly the
// lcp-intervals of the lexicographically sorted prompts (each branching
// point or prompt end at depth l is the maximal run of sorted prompts whose
// pairwise common prefix is >= l), and a node's hit count is the size of its
// interval.  So: sort the prompts, take the LCP of neighbours, and build the
// lcp-interval tree with one stack pass; each prompt's root path is the
// chain of intervals enclosing its position (plus its own leaf when it ends
// below no branching point).  A span is shared (hits >= 2) iff another
// prompt enters it, so a request's shared tokens are its longest common
// prefix with any other prompt.
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <limits>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "e2sched.h"

void e2_set_global_error(const char* m);

namespace {

struct ParseFail : std::runtime_error {
  using std::runtime_error::runtime_error;
};

[[noreturn]] void fail_at(const char* what, int64_t line, const std::string& detail) {
  throw ParseFail(std::string(what) + " line " + std::to_string(line) + ": " + detail);
}

int64_t to_int(const std::string& f, const char* what, int64_t line, const char* name) {
  int64_t v = 0;
  auto [p, ec] = std::from_chars(f.data(), f.data() + f.size(), v);
  if (ec != std::errc() || p != f.data() + f.size()) fail_at(what, line, std::string("bad ") + name + " '" + f + "'");
  return v;
}

double to_double(const std::string& f, const char* what, int64_t line, const char* name) {
  try {
    size_t used = 0;
    const double v = std::stod(f, &used);
    if (used == f.size()) return v;
  } catch (const std::exception&) {
  }
  fail_at(what, line, std::string("bad ") + name + " '" + f + "'");
}

std::string strip(const std::string& s) {
  const size_t b = s.find_first_not_of(" \t\r");
  if (b == std::string::npos) return "";
  return s.substr(b, s.find_last_not_of(" \t\r") - b + 1);
}

struct Corpus {
  std::vector<int32_t> tok;
  std::vector<int64_t> off{0};
  std::vector<int64_t> id, out;
  std::vector<double> arr;
  std::vector<int32_t> has_arr;
};

Corpus parse_corpus(std::istream& in) {
  Corpus c;
  std::string line, f;
  int64_t lineno = 0;
  std::vector<std::string> fields;
  while (std::getline(in, line)) {
    ++lineno;
    fields.clear();
    std::istringstream ls(line);
    while (ls >> f) fields.push_back(f);
    if (fields.empty()) continue;
    if (fields.size() < 3) fail_at("corpus", lineno, "expected id, tokens..., output_len");
    const int64_t id = to_int(fields[0], "corpus", lineno, "id");
    size_t k = 1;
    double arr = 0.0;
    int32_t has = 0;
    if (fields.size() >= 4 && fields[1].find('.') != std::string::npos) {
      arr = to_double(fields[1], "corpus", lineno, "arrival_ms");
      if (arr < 0.0) fail_at("corpus", lineno, "negative arrival_ms");
      has = 1;
      k = 2;
    }
    if (fields.size() - k < 2) fail_at("corpus", lineno, "prompt is empty");
    for (; k + 1 < fields.size(); ++k) {
      const int64_t t = to_int(fields[k], "corpus", lineno, "token id");
      if (t < std::numeric_limits<int32_t>::min() || t > std::numeric_limits<int32_t>::max())
        fail_at("corpus", lineno, "token id out of range '" + fields[k] + "'");
      c.tok.push_back((int32_t)t);
    }
    const int64_t out = to_int(fields.back(), "corpus", lineno, "output_len");
    if (out < 1) fail_at("corpus", lineno, "output_len must be >= 1");
    c.off.push_back((int64_t)c.tok.size());
    c.id.push_back(id);
    c.out.push_back(out);
    c.arr.push_back(arr);
    c.has_arr.push_back(has);
  }
  return c;
}

struct Row {
  double s;
  int64_t p, o;
};

std::vector<Row> parse_trace(std::istream& in) {
  std::string line;
  if (!std::getline(in, line)) throw ParseFail("trace line 1: missing header");
  {
    const std::string first = strip(line.substr(0, line.find(',')));
    char* end = nullptr;
    std::strtod(first.c_str(), &end);
    if (end != first.c_str() && *end == '\0') throw ParseFail("trace line 1: expected a header row, found data");
  }
  std::vector<Row> rows;
  int64_t lineno = 1;
  std::vector<std::string> fields;
  while (std::getline(in, line)) {
    ++lineno;
    if (strip(line).empty()) continue;
    fields.clear();
    size_t start = 0;
    for (;;) {
      const size_t comma = line.find(',', start);
      fields.push_back(strip(line.substr(start, comma == std::string::npos ? std::string::npos : comma - start)));
      if (comma == std::string::npos) break;
      start = comma + 1;
    }
    if (fields.size() != 3) fail_at("trace", lineno, "expected arrival_s, prompt_len, output_len");
    Row r;
    r.s = to_double(fields[0], "trace", lineno, "arrival_s");
    if (r.s < 0.0) fail_at("trace", lineno, "negative arrival_s");
    r.p = to_int(fields[1], "trace", lineno, "prompt_len");
    if (r.p < 1) fail_at("trace", lineno, "prompt_len must be >= 1");
    r.o = to_int(fields[2], "trace", lineno, "output_len");
    if (r.o < 1) fail_at("trace", lineno, "output_len must be >= 1");
    rows.push_back(r);
  }
  std::stable_sort(rows.begin(), rows.end(), [](const Row& a, const Row& b) { return a.s < b.s; });
  return rows;
}

e2_dist dist_of(std::vector<double> v) {
  e2_dist d;
  memset(&d, 0, sizeof(d));
  d.count = (int64_t)v.size();
  if (v.empty()) return d;
  std::sort(v.begin(), v.end());
  double sum = 0.0;
  for (double x : v) sum += x;
  d.mean = sum / (double)v.size();
  d.min = v.front();
  d.max = v.back();
  auto at = [&](double q) {
    int64_t r = (int64_t)std::ceil(q * (double)v.size());
    r = std::clamp<int64_t>(r, 1, (int64_t)v.size());
    return v[(size_t)(r - 1)];
  };
  d.p50 = at(0.50);
  d.p99 = at(0.99);
  return d;
}

// The corpus study over the lcp-interval tree of the sorted prompts.
void study(const int32_t* tok, const int64_t* off, const int64_t* outl, int64_t n, e2_study* rep) {
  memset(rep, 0, sizeof(*rep));
  rep->requests = n;
  if (n == 0) return;
  for (int64_t i = 0; i < n; ++i)
    if (off[i + 1] <= off[i]) throw std::invalid_argument("analyze: empty prompt");
  auto len = [&](int64_t i) { return off[i + 1] - off[i]; };
  // 1. sort the prompts; any byte-lexicographic order keeps every set of
  // prompts with a common token prefix contiguous
  std::vector<int64_t> sa((size_t)n);
  for (int64_t i = 0; i < n; ++i) sa[(size_t)i] = i;
  std::sort(sa.begin(), sa.end(), [&](int64_t a, int64_t b) {
    const int64_t la = len(a), lb = len(b);
    const int c = memcmp(tok + off[a], tok + off[b], (size_t)std::min(la, lb) * 4);
    return c != 0 ? c < 0 : (la != lb ? la < lb : a < b);
  });
  // 2. LCP of neighbours (lcp[k] between sa[k-1] and sa[k]; lcp[0] = lcp[n] = 0)
  std::vector<int64_t> lcp((size_t)n + 1, 0);
  for (int64_t k = 1; k < n; ++k) {
    const int64_t a = sa[(size_t)k - 1], b = sa[(size_t)k];
    const int64_t lim = std::min(len(a), len(b));
    const int32_t *pa = tok + off[a], *pb = tok + off[b];
    int64_t m = 0;
    while (m < lim && pa[m] == pb[m]) ++m;
    lcp[(size_t)k] = m;
  }
  // 3. lcp-interval tree: node 0 is the root (depth 0, all prompts)
  std::vector<int64_t> depth{0}, lb{0}, rb{n - 1};
  std::vector<int64_t> parent{-1};
  std::vector<int64_t> at((size_t)n + 1, 0);  // interval on top after boundary k
  std::vector<int64_t> st{0};
  for (int64_t k = 1; k <= n; ++k) {
    const int64_t v = k < n ? lcp[(size_t)k] : 0;
    int64_t start = k - 1, last = -1;
    while (v < depth[(size_t)st.back()]) {
      last = st.back();
      st.pop_back();
      rb[(size_t)last] = k - 1;
      start = lb[(size_t)last];
      if (v <= depth[(size_t)st.back()]) parent[(size_t)last] = st.back();
    }
    if (v > depth[(size_t)st.back()]) {
      const int64_t id = (int64_t)depth.size();
      depth.push_back(v);
      lb.push_back(start);
      rb.push_back(-1);
      parent.push_back(st.back());
      if (last >= 0) parent[(size_t)last] = id;
      st.push_back(id);
    }
    at[(size_t)k] = st.back();
  }
  // 4. per request, in corpus order
  std::vector<int64_t> pos((size_t)n);
  for (int64_t k = 0; k < n; ++k) pos[(size_t)sa[(size_t)k]] = k;
  std::vector<int64_t> chain;
  // key portions: interval id (>= 0) or ~position for a leaf of its own
  std::vector<std::pair<int64_t, std::pair<int64_t, int64_t>>> keys;
  std::vector<double> plens, olens;
  plens.reserve((size_t)n);
  olens.reserve((size_t)n);
  double shared_frac_sum = 0.0, ratio_sum = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t k = pos[(size_t)i], L = len(i);
    // deepest interval containing k: the deeper of its two boundaries
    const int64_t left = k > 0 ? at[(size_t)k] : 0, right = k + 1 < n ? at[(size_t)k + 1] : 0;
    int64_t deep = depth[(size_t)left] >= depth[(size_t)right] ? left : right;
    if (lcp[(size_t)k] == 0 && (k + 1 >= n || lcp[(size_t)k + 1] == 0)) deep = 0;
    chain.clear();
    for (int64_t x = deep; x > 0; x = parent[(size_t)x]) chain.push_back(x);
    std::reverse(chain.begin(), chain.end());
    // spans top-down: the intervals, then the prompt's own leaf below them
    const int64_t max_lcp = std::max(lcp[(size_t)k], k + 1 < n ? lcp[(size_t)k + 1] : 0);
    const int64_t shared = max_lcp;  // spans with hits >= 2 cover [0, max LCP)
    int64_t prefix = 0, key = 0, key_len = 0, key_hits = 0;
    bool have = false;
    int64_t s0 = 0;
    for (int64_t x : chain) {
      const int64_t m = depth[(size_t)x] - s0;
      if (m > prefix) {
        key = x;
        key_len = m;
        key_hits = rb[(size_t)x] - lb[(size_t)x] + 1;
        have = true;
      }
      prefix += m;
      s0 = depth[(size_t)x];
    }
    if (L > s0) {  // the prompt's own leaf (it ends below every branching point)
      const int64_t m = L - s0;
      if (m > prefix) {
        key = ~k;
        key_len = m;
        key_hits = 1;
        have = true;
      }
    }
    rep->total_prompt_tokens += L;
    rep->total_output_tokens += outl[i];
    rep->total_shared_tokens += shared;
    shared_frac_sum += (double)shared / (double)L;
    ratio_sum += (double)L / (double)outl[i];
    plens.push_back((double)L);
    olens.push_back((double)outl[i]);
    if (have) keys.push_back({key, {key_len, key_hits}});
  }
  const double dn = (double)n;
  rep->shared_token_fraction = (double)rep->total_shared_tokens / (double)rep->total_prompt_tokens;
  rep->mean_request_shared_fraction = shared_frac_sum / dn;
  rep->mean_prompt_output_ratio = ratio_sum / dn;
  rep->prompt_len = dist_of(std::move(plens));
  rep->output_len = dist_of(std::move(olens));
  std::sort(keys.begin(), keys.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
  keys.erase(std::unique(keys.begin(), keys.end(), [](const auto& a, const auto& b) { return a.first == b.first; }),
             keys.end());
  rep->key_portion_count = (int64_t)keys.size();
  std::vector<double> trav;
  double len_sum = 0.0;
  for (const auto& kv : keys) {
    len_sum += (double)kv.second.first;
    trav.push_back((double)kv.second.second);
  }
  if (!keys.empty()) rep->mean_key_portion_len = len_sum / (double)keys.size();
  rep->requests_per_shared_sequence = dist_of(std::move(trav));
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return E2_OK;
  } catch (const ParseFail& e) {
    e2_set_global_error(e.what());
    return E2_ERR_ARG;
  } catch (const std::exception& e) {
    e2_set_global_error(e.what());
    return E2_ERR_CONFIG;
  }
}

}  // namespace

extern "C" {

int e2_corpus_write(const char* path, const int32_t* tokens, const int64_t* offsets, const int64_t* ids,
                    const double* arrivals, const int32_t* has_arrival, const int64_t* output_lens, int64_t n) {
  return guarded([&] {
    std::ofstream out(path);
    if (!out) throw std::runtime_error(std::string("cannot open for writing: ") + path);
    char buf[40];
    std::string line;
    for (int64_t i = 0; i < n; ++i) {
      line = std::to_string(ids[i]);
      if (arrivals && (!has_arrival || has_arrival[i])) {
        std::snprintf(buf, sizeof(buf), "%.3f", arrivals[i]);
        line += ' ';
        line += buf;
      }
      for (int64_t k = offsets[i]; k < offsets[i + 1]; ++k) {
        line += ' ';
        line += std::to_string(tokens[k]);
      }
      line += ' ';
      line += std::to_string(output_lens[i]);
      line += '\n';
      out << line;
    }
    if (!out) throw std::runtime_error(std::string("write failed: ") + path);
  });
}

int e2_corpus_read(const char* path, int64_t* n, int64_t* n_tokens, int32_t* tokens, int64_t* offsets, int64_t* ids,
                   double* arrivals, int32_t* has_arrival, int64_t* output_lens) {
  return guarded([&] {
    std::ifstream in(path);
    if (!in) throw std::runtime_error(std::string("cannot open for reading: ") + path);
    const Corpus c = parse_corpus(in);
    *n = (int64_t)c.id.size();
    *n_tokens = (int64_t)c.tok.size();
    if (!tokens) return;
    std::copy(c.tok.begin(), c.tok.end(), tokens);
    std::copy(c.off.begin(), c.off.end(), offsets);
    std::copy(c.id.begin(), c.id.end(), ids);
    std::copy(c.arr.begin(), c.arr.end(), arrivals);
    std::copy(c.has_arr.begin(), c.has_arr.end(), has_arrival);
    std::copy(c.out.begin(), c.out.end(), output_lens);
  });
}

int e2_trace_read(const char* path, int64_t* n, double* arrival_s, int64_t* prompt_len, int64_t* output_len) {
  return guarded([&] {
    std::ifstream in(path);
    if (!in) throw std::runtime_error(std::string("cannot open for reading: ") + path);
    const std::vector<Row> rows = parse_trace(in);
    *n = (int64_t)rows.size();
    if (!arrival_s) return;
    for (size_t i = 0; i < rows.size(); ++i) {
      arrival_s[i] = rows[i].s;
      prompt_len[i] = rows[i].p;
      output_len[i] = rows[i].o;
    }
  });
}

int e2_synthesize_from_trace(const e2_workload_spec* content, uint64_t seed, const double* arrival_s,
                             const int64_t* prompt_len, const int64_t* output_len, int64_t n, int64_t* n_tokens,
                             int32_t* tokens, int64_t* offsets, int64_t* ids, double* arrivals_ms,
                             int64_t* output_lens) {
  return guarded([&] {
    const e2_workload_spec& s = *content;
    if (s.branch_count < 1) throw std::invalid_argument("workload: branch_count must be >= 1");
    if (s.zipf && s.zipf_s <= 0) throw std::invalid_argument("workload: zipf_s must be > 0");
    constexpr int64_t kSys = 1000000, kTrunk = 2000000, kFresh = 500000000, kIdMax = 2147483647;
    if (kSys + s.system_prompt_len > kIdMax || kTrunk + s.branch_count * s.branch_len > kIdMax)
      throw std::runtime_error("workload: token id space exhausted");
    std::vector<int64_t> order((size_t)n);
    for (int64_t i = 0; i < n; ++i) order[(size_t)i] = i;
    std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return arrival_s[a] < arrival_s[b]; });
    std::mt19937_64 rng(seed);
    const int nb = (int)s.branch_count;
    std::vector<double> cdf;
    if (s.zipf) {
      double acc = 0;
      for (int k = 1; k <= nb; ++k) {
        acc += std::pow((double)k, -s.zipf_s);
        cdf.push_back(acc);
      }
      for (double& c : cdf) c /= acc;
    }
    std::uniform_int_distribution<int> pick(0, nb - 1);
    int64_t fresh = kFresh, total = 0;
    std::vector<int32_t> p;
    for (int64_t j = 0; j < n; ++j) {
      const int64_t r = order[(size_t)j];
      int b;
      if (s.zipf) {
        const double u = std::uniform_real_distribution<double>(0.0, 1.0)(rng);
        b = (int)std::min<std::ptrdiff_t>(std::lower_bound(cdf.begin(), cdf.end(), u) - cdf.begin(), nb - 1);
      } else {
        b = pick(rng);
      }
      const int64_t want = prompt_len[r];
      p.clear();
      for (int64_t t = 0; t < s.system_prompt_len && (int64_t)p.size() < want; ++t) p.push_back((int32_t)(kSys + t));
      for (int64_t t = 0; t < s.branch_len && (int64_t)p.size() < want; ++t)
        p.push_back((int32_t)(kTrunk + (int64_t)b * s.branch_len + t));
      const int64_t rest = want - (int64_t)p.size();
      if (rest > 0) {
        if (fresh + rest > kIdMax) throw std::runtime_error("workload: token id space exhausted");
        for (int64_t t = 0; t < rest; ++t) p.push_back((int32_t)(fresh++));
      }
      if (tokens) {
        std::copy(p.begin(), p.end(), tokens + total);
        offsets[j] = total;
        offsets[j + 1] = total + (int64_t)p.size();
        ids[j] = j + 1;
        arrivals_ms[j] = arrival_s[r] * 1000.0;
        output_lens[j] = output_len[r];
      }
      total += (int64_t)p.size();
    }
    *n_tokens = total;
  });
}

int e2_analyze(const int32_t* tokens, const int64_t* offsets, const int64_t* output_lens, int64_t n, e2_study* out) {
  return guarded([&] { study(tokens, offsets, output_lens, n, out); });
}

}  // extern "C"
