// K1: cost model + task divider + LPT schedule, host C++ (float64).
//
// Bit-exact restatement of reference prefixdec/cost_model.py:56-84 and
// prefixdec/scheduler.py:81-242. Exactness rules:
//   * same association order of every float64 expression; the library is
//     built with -ffp-contract=off so a*b+c is never fused;
//   * log2 comes from the same libm as CPython's math.log2;
//   * the reference's builtin sum() over floats is CPython >= 3.12's
//     Neumaier-compensated sum (bltinmodule.c), reproduced in py_sum();
//   * LPT order (-cost, index), block choice (load, block), grid-search key
//     (makespan, #subtasks, b_k) with first-minimum tie breaking.
// The grid search additionally prunes candidates whose makespan lower
// bound already exceeds the best found; pruning never changes the winner
// because a candidate with a larger makespan can never have a smaller key.
#include <algorithm>
#include <cmath>
#include <limits>
#include <queue>
#include <string>
#include <vector>

#include "common.h"

using codec::fail;

namespace {

struct Table {
  const codec_cost_table* t;
  int64_t nq(int i) const { return t->nq_knots[i]; }
  int64_t n(int i) const { return t->n_knots[i]; }
  double cost(int ni, int qi) const { return t->cost_ms[(int64_t)ni * t->n_nq + qi]; }
};

// Clamped bracket (cost_model.py:56-65)
inline void segment(const int64_t* knots, int32_t cnt, int64_t x, int32_t& lo, int32_t& hi) {
  if (x <= knots[0]) {
    lo = hi = 0;
    return;
  }
  if (x >= knots[cnt - 1]) {
    lo = hi = cnt - 1;
    return;
  }
  int32_t h = 1;
  while (knots[h] < x) ++h;
  lo = h - 1;
  hi = h;
}

double estimate(const codec_cost_table* t, int64_t n_q, int64_t n) {
  int32_t a, b, c, d;
  segment(t->nq_knots, t->n_nq, n_q, a, b);
  double tq = 0.0;
  if (a != b) tq = (double)(n_q - t->nq_knots[a]) / (double)(t->nq_knots[b] - t->nq_knots[a]);
  segment(t->n_knots, t->n_n, n, c, d);
  double tn = 0.0;
  if (c != d) {
    double la = std::log2((double)t->n_knots[c]);
    double lb = std::log2((double)t->n_knots[d]);
    tn = (std::log2((double)n) - la) / (lb - la);
  }
  const double* g = t->cost_ms;
  const int32_t w = t->n_nq;
  double c00 = g[(int64_t)c * w + a], c01 = g[(int64_t)c * w + b];
  double c10 = g[(int64_t)d * w + a], c11 = g[(int64_t)d * w + b];
  double low = c00 + tq * (c01 - c00);
  double high = c10 + tq * (c11 - c10);
  return low + tn * (high - low);
}

// CPython >= 3.12 builtin sum() over floats with int start 0.
struct PySum {
  bool any = false;
  double total = 0.0, comp = 0.0;
  inline void add(double x) {
    if (!any) {
      total = x;  // 0 + x is exact
      any = true;
      return;
    }
    double t = total + x;
    if (std::fabs(total) >= std::fabs(x))
      comp += (total - t) + x;
    else
      comp += (x - t) + total;
    total = t;
  }
  inline double result() const {
    double r = total;
    if (comp != 0.0 && std::isfinite(comp)) r += comp;
    return r;
  }
};

inline int64_t clamp_b(int64_t n, int64_t b) { return std::max<int64_t>(1, std::min(b, n)); }
inline int64_t slice_step(int64_t n, int64_t b) {
  b = clamp_b(n, b);
  return (n + b - 1) / b;
}
inline int64_t canonical(int64_t n, int64_t b) {
  int64_t s = slice_step(n, b);
  return (n + s - 1) / s;
}

// ceil(x) as the slice request of lower_bound / caps; values past n are
// all equivalent after slice_ranges clamps them.
inline int64_t ceil_req(double x) {
  double c = std::ceil(x);
  if (!(c < 9.0e18)) return std::numeric_limits<int64_t>::max() / 4;
  return (int64_t)c;
}

double sliced_volume(const codec_cost_table* t, int64_t nq, int64_t n, int64_t b) {
  int64_t step = slice_step(n, b);
  PySum s;
  double full = estimate(t, nq, step);
  int64_t k = 0;
  for (int64_t start = 0; start < n; start += step, ++k) {
    int64_t stop = std::min(start + step, n);
    s.add(stop - start == step ? full : estimate(t, nq, stop - start));
  }
  return s.result();
}

double lower_bound(const codec_cost_table* t, int32_t nt, const int64_t* nq, const int64_t* n,
                   int32_t m, double tol) {
  std::vector<double> full(nt);
  PySum hs;
  double lo = -std::numeric_limits<double>::infinity();
  for (int32_t j = 0; j < nt; ++j) {
    full[j] = estimate(t, nq[j], n[j]);
    hs.add(full[j]);
  }
  for (int32_t j = 0; j < nt; ++j) lo = std::max(lo, estimate(t, nq[j], 1));
  double hi = hs.result();
  auto ok = [&](double c) {
    double vol = 0.0;
    for (int32_t j = 0; j < nt; ++j) vol += sliced_volume(t, nq[j], n[j], ceil_req(full[j] / c));
    return vol / (double)m <= c;
  };
  if (ok(lo)) return lo;
  while (hi - lo > tol) {
    double mid = 0.5 * (lo + hi);
    if (ok(mid))
      hi = mid;
    else
      lo = mid;
  }
  return hi;
}

// LPT (scheduler.py:142-155): returns makespan; fills owner/loads if given.
struct Lpt {
  std::vector<int32_t> order;
  std::vector<double> loads;
  double run(const std::vector<double>& costs, int32_t m, int32_t* owner, double* loads_out,
             double prune_above) {
    const int64_t S = (int64_t)costs.size();
    order.resize(S);
    for (int64_t i = 0; i < S; ++i) order[i] = (int32_t)i;
    std::stable_sort(order.begin(), order.end(), [&](int32_t x, int32_t y) {
      double cx = -costs[x], cy = -costs[y];
      if (cx < cy) return true;
      if (cy < cx) return false;
      return x < y;
    });
    loads.assign(m, 0.0);
    // min-heap on (load, block)
    using E = std::pair<double, int32_t>;
    std::priority_queue<E, std::vector<E>, std::greater<E>> heap;
    for (int32_t j = 0; j < m; ++j) heap.push({0.0, j});
    double mk = 0.0;
    for (int64_t k = 0; k < S; ++k) {
      int32_t i = order[k];
      E top = heap.top();
      heap.pop();
      int32_t b = top.second;
      loads[b] += costs[i];
      if (owner) owner[i] = b;
      heap.push({loads[b], b});
      if (loads[b] > mk) mk = loads[b];
      if (mk > prune_above) return mk;  // cannot win; caller discards
    }
    if (loads_out) std::copy(loads.begin(), loads.end(), loads_out);
    mk = loads.empty() ? 0.0 : *std::max_element(loads.begin(), loads.end());
    return mk;
  }
};

}  // namespace

struct codec_plan {
  int32_t blocks = 0;
  bool truncated = false;
  double makespan = 0.0, cost_l = std::numeric_limits<double>::quiet_NaN();
  std::vector<int64_t> b_k;
  std::vector<int32_t> sub_task, block_of;
  std::vector<int64_t> sub_node, sub_start, sub_stop;
  std::vector<double> sub_cost, loads;
};

namespace {

// _plan_for (scheduler.py:158-180): canonical b_k, expand, LPT
codec_plan* plan_for(const codec_cost_table* t, int32_t nt, const int64_t* node, const int64_t* nq,
                     const int64_t* n, const int64_t* bk_req, int32_t m, double cost_l, bool truncated) {
  auto p = new codec_plan();
  p->blocks = m;
  p->truncated = truncated;
  p->cost_l = cost_l;
  p->b_k.resize(nt);
  for (int32_t j = 0; j < nt; ++j) {
    int64_t b = canonical(n[j], bk_req[j]);
    p->b_k[j] = b;
    int64_t step = slice_step(n[j], b);
    for (int64_t s = 0; s < n[j]; s += step) {
      int64_t e = std::min(s + step, n[j]);
      p->sub_task.push_back(j);
      p->sub_node.push_back(node[j]);
      p->sub_start.push_back(s);
      p->sub_stop.push_back(e);
      p->sub_cost.push_back(estimate(t, nq[j], e - s));
    }
  }
  p->block_of.assign(p->sub_cost.size(), 0);
  p->loads.assign(m, 0.0);
  Lpt lpt;
  p->makespan = lpt.run(p->sub_cost, m, p->block_of.data(), p->loads.data(),
                        std::numeric_limits<double>::infinity());
  return p;
}

bool valid_table(const codec_cost_table* t) {
  return t && t->n_nq >= 1 && t->n_n >= 1 && t->nq_knots && t->n_knots && t->cost_ms;
}

}  // namespace

extern "C" double codec_estimate(const codec_cost_table* t, int64_t n_q, int64_t n) {
  if (!valid_table(t)) return std::numeric_limits<double>::quiet_NaN();
  return estimate(t, n_q, n);
}

extern "C" int32_t codec_slice_ranges(int64_t n, int64_t b, int64_t* start_stop, int64_t cap,
                                      int64_t* count) {
  if (n < 1) return fail(CODEC_ERR_VALUE, "slice_ranges needs n >= 1, got %lld", (long long)n);
  int64_t step = slice_step(n, b);
  int64_t k = 0;
  for (int64_t s = 0; s < n; s += step, ++k) {
    if (start_stop && k < cap) {
      start_stop[2 * k] = s;
      start_stop[2 * k + 1] = std::min(s + step, n);
    }
  }
  if (count) *count = k;
  return CODEC_OK;
}

extern "C" int32_t codec_lower_bound(const codec_cost_table* t, int32_t n_tasks, const int64_t* task_nq,
                                     const int64_t* task_n, int32_t m, double tol, double* cost_l) {
  if (!valid_table(t)) return fail(CODEC_ERR_VALUE, "invalid cost table");
  if (n_tasks < 1) return fail(CODEC_ERR_VALUE, "no tasks to schedule");
  if (m < 1) return fail(CODEC_ERR_VALUE, "need m >= 1 blocks, got %d", m);
  *cost_l = lower_bound(t, n_tasks, task_nq, task_n, m, tol);
  return CODEC_OK;
}

extern "C" int32_t codec_division_caps(const codec_cost_table* t, int32_t n_tasks, const int64_t* task_nq,
                                       const int64_t* task_n, double cost_l, int64_t* caps) {
  if (!valid_table(t)) return fail(CODEC_ERR_VALUE, "invalid cost table");
  if (!(cost_l > 0)) return fail(CODEC_ERR_VALUE, "cost_l must be positive, got %.17g", cost_l);
  for (int32_t j = 0; j < n_tasks; ++j) caps[j] = ceil_req(estimate(t, task_nq[j], task_n[j]) / cost_l);
  return CODEC_OK;
}

extern "C" int32_t codec_greedy_assign(int64_t n, const double* costs, int32_t m, int32_t* block_of,
                                       double* loads) {
  if (m < 1) return fail(CODEC_ERR_VALUE, "need m >= 1 blocks, got %d", m);
  std::vector<double> c(costs, costs + n);
  Lpt lpt;
  lpt.run(c, m, block_of, loads, std::numeric_limits<double>::infinity());
  return CODEC_OK;
}

extern "C" int32_t codec_divide_and_schedule(const codec_cost_table* t, int32_t nt, const int64_t* node,
                                             const int64_t* nq, const int64_t* n, int32_t m,
                                             int64_t search_limit, int32_t on_overflow, codec_plan** out) {
  if (!out) return fail(CODEC_ERR_VALUE, "out handle is NULL");
  *out = nullptr;
  if (!valid_table(t)) return fail(CODEC_ERR_VALUE, "invalid cost table");
  if (nt < 1) return fail(CODEC_ERR_VALUE, "no tasks to schedule");
  if (m < 1) return fail(CODEC_ERR_VALUE, "need m >= 1 blocks, got %d", m);
  for (int32_t j = 0; j < nt; ++j)
    if (n[j] < 1 || nq[j] < 1)
      return fail(CODEC_ERR_VALUE, "task (%lld, %lld) must have n, n_q >= 1", (long long)nq[j], (long long)n[j]);

  const double cost_l = lower_bound(t, nt, nq, n, m, 1e-4);
  // options: sorted distinct canonical divisions up to the cap
  std::vector<std::vector<int64_t>> options(nt);
  unsigned __int128 total = 1;
  bool total_overflow = false;
  const unsigned __int128 sat = (unsigned __int128)1 << 100;
  for (int32_t j = 0; j < nt; ++j) {
    int64_t cap = ceil_req(estimate(t, nq[j], n[j]) / cost_l);
    int64_t hi = std::max<int64_t>(1, std::min(cap, n[j]));
    std::vector<int64_t>& o = options[j];
    // canonical_division(n, b) is non-increasing in step, i.e. walk b and dedupe
    int64_t last = -1;
    for (int64_t b = 1; b <= hi; ++b) {
      int64_t cnt = canonical(n[j], b);
      if (cnt != last) {
        o.push_back(cnt);
        last = cnt;
      }
      // jump to the next b that changes the step
      int64_t step = slice_step(n[j], b);
      if (step > 1) {
        // smallest b' with ceil(n/b') < step  <=>  b' > (n-1)/(step-1)
        int64_t nb = (n[j] - 1) / (step - 1) + 1;
        if (nb - 1 > b) b = std::min(nb - 1, hi);
      }
    }
    std::sort(o.begin(), o.end());
    o.erase(std::unique(o.begin(), o.end()), o.end());
    if (!total_overflow) {
      total *= (unsigned __int128)o.size();
      if (total > sat) total_overflow = true;
    }
  }
  bool over = total_overflow || total > (unsigned __int128)(search_limit < 0 ? 0 : search_limit);
  if (over && on_overflow == 1) {
    std::string tot;
    if (total_overflow) {
      tot = "> 2**100";
    } else {
      unsigned __int128 v = total;
      if (v == 0) tot = "0";
      while (v > 0) {
        tot.insert(tot.begin(), char('0' + (int)(v % 10)));
        v /= 10;
      }
    }
    return fail(CODEC_ERR_SEARCH_SPACE_OVERFLOW, "%s division candidates exceed the limit of %lld",
                tot.c_str(), (long long)search_limit);
  }

  std::vector<int64_t> best_bk;
  double best_mk = std::numeric_limits<double>::infinity();
  int64_t best_ns = 0;
  bool have = false;

  // Evaluating a candidate only needs its makespan (the key's first term;
  // #subtasks and b_k are free). LPT's load multiset -- hence the makespan,
  // bit for bit -- depends only on the descending cost sequence: items of
  // equal cost are interchangeable and equal-load blocks are symmetric.
  // So tasks with a single option are expanded and sorted once, varying
  // tasks per candidate, and the two sorted runs are merged into a
  // load-only min-heap. The exact owner/index tie-breaks are applied once,
  // to the winner, by plan_for().
  std::vector<double> fixed_costs;
  std::vector<int32_t> varying;
  double fixed_sum = 0.0, fixed_max = 0.0;
  int64_t fixed_ns = 0;
  for (int32_t j = 0; j < nt; ++j) {
    if (options[j].size() > 1 && !over) {
      varying.push_back(j);
      continue;
    }
    // over: both candidates are evaluated with the generic path below
    if (over) continue;
    int64_t step = slice_step(n[j], options[j][0]);
    double cfull = estimate(t, nq[j], step);
    for (int64_t s = 0; s < n[j]; s += step) {
      int64_t e = std::min(s + step, n[j]);
      double c = (e - s == step) ? cfull : estimate(t, nq[j], e - s);
      fixed_costs.push_back(c);
      fixed_sum += c;
      fixed_max = std::max(fixed_max, c);
      ++fixed_ns;
    }
  }
  std::sort(fixed_costs.begin(), fixed_costs.end(), std::greater<double>());
  std::vector<double> var_costs;
  std::vector<double> heap;
  std::vector<int64_t> bk_c(nt);

  auto lpt_makespan = [&](double prune_above) {
    // merge the two descending runs into a min-heap of block loads
    heap.assign(m, 0.0);  // all zeros is a valid min-heap
    double mk = 0.0;
    size_t a = 0, b = 0;
    const size_t na = fixed_costs.size(), nb = var_costs.size();
    while (a < na || b < nb) {
      double c;
      if (b >= nb || (a < na && fixed_costs[a] >= var_costs[b]))
        c = fixed_costs[a++];
      else
        c = var_costs[b++];
      std::pop_heap(heap.begin(), heap.end(), std::greater<double>());
      double nl = heap.back() + c;
      heap.back() = nl;
      std::push_heap(heap.begin(), heap.end(), std::greater<double>());
      if (nl > mk) mk = nl;
      if (mk > prune_above) return mk;
    }
    return mk;
  };

  auto eval = [&](const std::vector<int64_t>& bk_in) {
    for (int32_t j = 0; j < nt; ++j) bk_c[j] = canonical(n[j], bk_in[j]);
    const std::vector<int64_t>& bk = bk_c;
    var_costs.clear();
    double vmax = fixed_max, vsum = 0.0;
    int64_t ns = fixed_ns;
    const bool all = over;  // fallback candidates: every task is "varying"
    auto add_task = [&](int32_t j) {
      int64_t step = slice_step(n[j], bk[j]);
      double cfull = estimate(t, nq[j], step);
      for (int64_t s = 0; s < n[j]; s += step) {
        int64_t e = std::min(s + step, n[j]);
        double c = (e - s == step) ? cfull : estimate(t, nq[j], e - s);
        var_costs.push_back(c);
        vmax = std::max(vmax, c);
        vsum += c;
        ++ns;
      }
    };
    if (all)
      for (int32_t j = 0; j < nt; ++j) add_task(j);
    else
      for (int32_t j : varying) add_task(j);
    // lower bound on the LPT makespan: largest item and average load (a
    // 1e-9 relative guard keeps the float comparison conservative)
    if (have) {
      double lb = std::max(vmax, (fixed_sum + vsum) / (double)m);
      if (lb * (1.0 - 1e-9) > best_mk) return;
    }
    std::sort(var_costs.begin(), var_costs.end(), std::greater<double>());
    double mk = lpt_makespan(have ? best_mk : std::numeric_limits<double>::infinity());
    bool better;
    if (!have) {
      better = true;
    } else if (mk != best_mk) {
      better = mk < best_mk;
    } else if (ns != best_ns) {
      better = ns < best_ns;
    } else {
      better = bk < best_bk;
    }
    if (better) {
      have = true;
      best_mk = mk;
      best_ns = ns;
      best_bk = bk;
    }
  };

  if (over) {
    std::vector<int64_t> ident(nt, 1), capd(nt);
    for (int32_t j = 0; j < nt; ++j) capd[j] = options[j].back();
    // canonicalise like _plan_for before comparing keys
    eval(ident);
    eval(capd);
  } else {
    std::vector<size_t> pos(nt, 0);
    std::vector<int64_t> bk(nt);
    for (int32_t j = 0; j < nt; ++j) bk[j] = options[j][0];
    while (true) {
      eval(bk);
      int32_t j = nt - 1;
      while (j >= 0) {
        if (++pos[j] < options[j].size()) {
          bk[j] = options[j][pos[j]];
          break;
        }
        pos[j] = 0;
        bk[j] = options[j][0];
        --j;
      }
      if (j < 0) break;
    }
  }
  *out = plan_for(t, nt, node, nq, n, best_bk.data(), m, cost_l, over);
  return CODEC_OK;
}

extern "C" int32_t codec_plan_uniform(const codec_cost_table* t, int32_t nt, const int64_t* node,
                                      const int64_t* nq, const int64_t* n, int32_t m, int64_t bk,
                                      double cost_l, codec_plan** out) {
  if (!out) return fail(CODEC_ERR_VALUE, "out handle is NULL");
  *out = nullptr;
  if (!valid_table(t)) return fail(CODEC_ERR_VALUE, "invalid cost table");
  if (bk < 1) return fail(CODEC_ERR_VALUE, "b_k must be >= 1, got %lld", (long long)bk);
  if (m < 1) return fail(CODEC_ERR_VALUE, "need m >= 1 blocks, got %d", m);
  std::vector<int64_t> req(nt, bk);
  *out = plan_for(t, nt, node, nq, n, req.data(), m, cost_l, false);
  return CODEC_OK;
}

extern "C" void codec_plan_free(codec_plan* p) { delete p; }

extern "C" int32_t codec_plan_info_get(const codec_plan* p, codec_plan_info* info) {
  if (!p || !info) return fail(CODEC_ERR_VALUE, "NULL argument");
  info->n_tasks = (int32_t)p->b_k.size();
  info->n_subtasks = (int32_t)p->sub_task.size();
  info->blocks = p->blocks;
  info->truncated = p->truncated ? 1 : 0;
  info->makespan_ms = p->makespan;
  info->cost_l_ms = p->cost_l;
  return CODEC_OK;
}

extern "C" int32_t codec_plan_read(const codec_plan* p, int64_t* b_k, int32_t* sub_task, int64_t* sub_node,
                                   int64_t* sub_start, int64_t* sub_stop, double* sub_cost, int32_t* block_of,
                                   double* loads) {
  if (!p) return fail(CODEC_ERR_VALUE, "NULL plan");
  if (b_k) std::copy(p->b_k.begin(), p->b_k.end(), b_k);
  if (sub_task) std::copy(p->sub_task.begin(), p->sub_task.end(), sub_task);
  if (sub_node) std::copy(p->sub_node.begin(), p->sub_node.end(), sub_node);
  if (sub_start) std::copy(p->sub_start.begin(), p->sub_start.end(), sub_start);
  if (sub_stop) std::copy(p->sub_stop.begin(), p->sub_stop.end(), sub_stop);
  if (sub_cost) std::copy(p->sub_cost.begin(), p->sub_cost.end(), sub_cost);
  if (block_of) std::copy(p->block_of.begin(), p->block_of.end(), block_of);
  if (loads) std::copy(p->loads.begin(), p->loads.end(), loads);
  return CODEC_OK;
}

// merge_schedule() / sequential_schedule() (executor.py:86-117): the
// reference's per-request combination order of partials numbered 0..P-1 in
// path-then-slice order. Balanced: each round pairs adjacent survivors,
// the left label survives (ceil(log2 P) rounds); sequential: P-1 rounds of
// (0, i). The device merge (kern_merge.cu) folds all P at once in one pass
// -- equal up to rounding (test_attention.py:160-180); the schedule is the
// reference's integer contract.
extern "C" int32_t codec_merge_schedule(int32_t mode, int64_t path_len, const int64_t* slices_per_node,
                                        int64_t n_counts, int64_t* pairs, int64_t* round_ptr, int64_t cap,
                                        int64_t* n_pairs, int64_t* n_rounds) {
  if (!n_pairs || !n_rounds) return codec::fail(CODEC_ERR_VALUE, "NULL argument");
  int64_t total = 0;
  if (mode == 0) {
    if (path_len < 1) return codec::fail(CODEC_ERR_VALUE, "path_len must be >= 1");
    if (n_counts != path_len)
      return codec::fail(CODEC_ERR_VALUE, "expected %lld per-node slice counts, got %lld", (long long)path_len,
                         (long long)n_counts);
    for (int64_t i = 0; i < n_counts; ++i) total += slices_per_node[i];
  } else if (mode == 1) {
    total = path_len;  // sequential_schedule(total)
  } else {
    return codec::fail(CODEC_ERR_VALUE, "mode must be 0 (balanced) or 1 (sequential)");
  }
  std::vector<int64_t> out_pairs, out_ptr{0};
  if (mode == 1) {
    for (int64_t i = 1; i < total; ++i) {
      out_pairs.push_back(0);
      out_pairs.push_back(i);
      out_ptr.push_back((int64_t)out_pairs.size() / 2);
    }
  } else {
    std::vector<int64_t> labels(total > 0 ? total : 0);
    for (int64_t i = 0; i < total; ++i) labels[i] = i;
    while (labels.size() > 1) {
      std::vector<int64_t> next;
      for (size_t i = 0; i + 1 < labels.size(); i += 2) {
        out_pairs.push_back(labels[i]);
        out_pairs.push_back(labels[i + 1]);
        next.push_back(labels[i]);
      }
      if (labels.size() % 2) next.push_back(labels.back());
      out_ptr.push_back((int64_t)out_pairs.size() / 2);
      labels.swap(next);
    }
  }
  *n_pairs = (int64_t)out_pairs.size() / 2;
  *n_rounds = (int64_t)out_ptr.size() - 1;
  if (pairs && round_ptr) {
    if (cap < *n_pairs) return codec::fail(CODEC_ERR_VALUE, "pair buffer holds %lld of %lld", (long long)cap,
                                           (long long)*n_pairs);
    std::copy(out_pairs.begin(), out_pairs.end(), pairs);
    std::copy(out_ptr.begin(), out_ptr.end(), round_ptr);
  }
  return CODEC_OK;
}
