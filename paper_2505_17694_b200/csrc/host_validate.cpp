// Host-side structural checks that report instead of raising:
//   * codec_forest_validate -- every invariant of a (possibly corrupted)
//     forest snapshot, the contract of the reference's validate()
//     (forest.py:266-363): same violation codes, same messages, same order;
//   * codec_cost_grid / codec_cost_table_check -- profile rows to a dense
//     (n, n_q) grid and the CostTable invariants (load_profile /
//     CostTable.__post_init__, cost_model.py:39-53, :102-150).
// The Python layer (forest.validate, cost_model.load_profile) marshals the
// objects into flat arrays and turns the records back into Violation /
// exception objects.
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <map>
#include <set>
#include <sstream>
#include <string>
#include <utility>
#include <vector>

#include "common.h"

using codec::fail;

namespace {

// Python repr of a tuple of ints: (), (a,), (a, b, ...)
std::string py_tuple(const int64_t* v, int64_t n) {
  std::ostringstream os;
  os << "(";
  for (int64_t i = 0; i < n; ++i) os << (i ? ", " : "") << v[i];
  if (n == 1) os << ",";
  os << ")";
  return os.str();
}

// Python repr of a float: the shortest round-tripping %g, ".0" on integers
std::string py_float(double x) {
  char buf[64];
  for (int p = 1; p <= 17; ++p) {
    snprintf(buf, sizeof(buf), "%.*g", p, x);
    if (strtod(buf, nullptr) == x || x != x) break;
  }
  std::string s = buf;
  if (s.find_first_of(".eEni") == std::string::npos) s += ".0";
  return s;
}

constexpr int64_t kNone = INT64_MIN;  // Violation field None (-1 is a request id a corrupted query set may hold)

struct Rec {
  int32_t code;
  int64_t node, request;  // kNone: None
  std::string msg;
};

}  // namespace

struct codec_report {
  std::vector<Rec> recs;
};

extern "C" int32_t codec_forest_validate(int32_t n_nodes, const int64_t* node_id, const int64_t* parent,
                                         const int64_t* length, const int32_t* kv_state, const int64_t* kv_tail_ptr,
                                         const int64_t* kv_tail, int64_t h_kv, int64_t d,
                                         const int64_t* children_ptr, const int64_t* children_idx, int32_t bs,
                                         const int64_t* path_ptr, const int64_t* path_idx, const int64_t* qset_ptr,
                                         const int64_t* qset_idx, int64_t n_vis, const int64_t* vis_node,
                                         const int64_t* vis_req, const int64_t* vis_count,
                                         const int64_t* token_offset, int64_t n_token_offset, codec_report** out) {
  if (!out) return fail(CODEC_ERR_VALUE, "NULL argument");
  *out = nullptr;
  if (n_nodes < 0 || bs < 0) return fail(CODEC_ERR_VALUE, "negative sizes");
  auto rep = new codec_report();
  auto& R = rep->recs;
  auto add = [&](int32_t code, int64_t node, int64_t req, std::string msg) {
    R.push_back({code, node, req, std::move(msg)});
  };
  const int64_t N = n_nodes;
  auto in_nodes = [&](int64_t x) { return x >= 0 && x < N; };
  auto path_of = [&](int64_t r) { return std::make_pair(path_idx + path_ptr[r], path_ptr[r + 1] - path_ptr[r]); };

  // ids are positions
  for (int64_t i = 0; i < N; ++i)
    if (node_id[i] != i) add(CODEC_VIOLATION_BAD_NODE_INDEX, i, kNone, "nodes[" + std::to_string(i) + "] has id " +
                                                                          std::to_string(node_id[i]));
  if (N > 0 && length[0] != 0) add(CODEC_VIOLATION_NON_EMPTY_ROOT, 0, kNone, "virtual root must hold no tokens");
  // per node: tokens, then K/V shapes (kv_state: 0 not checked / fine,
  // 1 K and V shapes differ, 2 keys.shape[1:] given in kv_tail)
  for (int64_t i = 1; i < N; ++i) {
    const std::string nid = std::to_string(node_id[i]);
    if (length[i] < 1) add(CODEC_VIOLATION_EMPTY_NON_ROOT, node_id[i], kNone, "node " + nid + " has len 0");
    if (kv_state[i] == 1) {
      add(CODEC_VIOLATION_DIMENSION_MISMATCH, node_id[i], kNone, "node " + nid + " K/V shapes differ");
    } else if (kv_state[i] == 2) {
      const int64_t* tail = kv_tail + kv_tail_ptr[i];
      const int64_t nt = kv_tail_ptr[i + 1] - kv_tail_ptr[i];
      if (!(nt == 2 && tail[0] == h_kv && tail[1] == d))
        add(CODEC_VIOLATION_DIMENSION_MISMATCH, node_id[i], kNone,
            "node " + nid + " is " + py_tuple(tail, nt) + ", forest is (" + std::to_string(h_kv) + ", " +
                std::to_string(d) + ")");
    }
  }
  // parent links reach the root without repeating a node
  for (int64_t i = 1; i < N; ++i) {
    std::set<int64_t> seen{node_id[i]};
    int64_t cur = parent[i];
    bool ok = true;
    while (cur != 0) {
      if (seen.count(cur) || !in_nodes(cur)) {
        add(CODEC_VIOLATION_CYCLE_DETECTED, node_id[i], kNone,
            "parent chain of node " + std::to_string(node_id[i]) + " never reaches root");
        ok = false;
        break;
      }
      seen.insert(cur);
      cur = parent[cur];
    }
    if (ok && parent[i] >= N)
      add(CODEC_VIOLATION_DANGLING_PARENT, node_id[i], kNone,
          "node " + std::to_string(node_id[i]) + " parent " + std::to_string(parent[i]) + " missing");
  }
  // children lists vs parent fields, as sets of (parent, child) edges
  {
    std::set<std::pair<int64_t, int64_t>> adj, decl;
    for (int64_t i = 0; i < N; ++i)
      for (int64_t j = children_ptr[i]; j < children_ptr[i + 1]; ++j) {
        const int64_t c = children_idx[j];
        if (!in_nodes(c)) {
          delete rep;
          return fail(CODEC_ERR_VALUE, "children list names node %lld outside the forest", (long long)c);
        }
        adj.insert({parent[c], c});
      }
    for (int64_t i = 1; i < N; ++i) decl.insert({parent[i], node_id[i]});
    if (adj != decl) add(CODEC_VIOLATION_ADJACENCY_MISMATCH, kNone, kNone, "children lists disagree with parent fields");
  }
  // request paths are parent -> child chains from the root
  for (int64_t r = 0; r < bs; ++r) {
    auto [p, n] = path_of(r);
    int64_t prev = 0;
    for (int64_t k = 0; k < n; ++k) {
      const int64_t x = p[k];
      if (!(x >= 1 && x < N) || parent[x] != prev) {
        add(CODEC_VIOLATION_PATH_NOT_PREFIX_CHAIN, kNone, r,
            "request " + std::to_string(r) + " path " + py_tuple(p, n) + " breaks at " + std::to_string(x));
        break;
      }
      prev = x;
    }
  }
  // r in I_n  <=>  n on path(r), query sets ascending
  auto on_path = [&](int64_t r, int64_t nid) {
    auto [p, n] = path_of(r);
    return std::find(p, p + n, nid) != p + n;
  };
  for (int64_t i = 1; i < N; ++i) {
    const int64_t* qs = qset_idx + qset_ptr[i];
    const int64_t nq = qset_ptr[i + 1] - qset_ptr[i];
    std::vector<int64_t> srt(qs, qs + nq);
    std::sort(srt.begin(), srt.end());
    srt.erase(std::unique(srt.begin(), srt.end()), srt.end());
    if (!std::equal(qs, qs + nq, srt.begin(), srt.end()))
      add(CODEC_VIOLATION_QUERY_SET_UNSORTED, node_id[i], kNone,
          "node " + std::to_string(node_id[i]) + " query_set not ascending");
    for (int64_t k = 0; k < nq; ++k) {
      int64_t rid = qs[k];
      bool bad = rid >= bs;
      if (!bad) {
        if (rid < -(int64_t)bs) {
          delete rep;
          return fail(CODEC_ERR_VALUE, "query_set of node %lld names request %lld", (long long)node_id[i],
                      (long long)rid);
        }
        bad = !on_path(rid < 0 ? rid + bs : rid, node_id[i]);  // Python's negative index
      }
      if (bad)
        add(CODEC_VIOLATION_QUERY_SET_PATH_MISMATCH, node_id[i], rid,
            "node " + std::to_string(node_id[i]) + " lists request " + std::to_string(rid) + " whose path misses it");
    }
  }
  for (int64_t r = 0; r < bs; ++r) {
    auto [p, n] = path_of(r);
    for (int64_t k = 0; k < n; ++k) {
      const int64_t x = p[k];
      if (!in_nodes(x)) continue;
      const int64_t* qs = qset_idx + qset_ptr[x];
      const int64_t nq = qset_ptr[x + 1] - qset_ptr[x];
      if (std::find(qs, qs + nq, r) == qs + nq)
        add(CODEC_VIOLATION_QUERY_SET_PATH_MISMATCH, x, r,
            "request " + std::to_string(r) + " runs through node " + std::to_string(x) +
                " but is not in its query_set");
    }
  }
  // visible counts within 1..len (entries in node order, then insertion order)
  for (int64_t e = 0; e < n_vis; ++e) {
    const int64_t x = vis_node[e];
    if (!(x >= 1 && x < N)) continue;
    if (!(vis_count[e] >= 1 && vis_count[e] <= length[x]))
      add(CODEC_VIOLATION_VISIBLE_LEN_OUT_OF_RANGE, node_id[x], vis_req[e],
          "node " + std::to_string(node_id[x]) + " visible_len[" + std::to_string(vis_req[e]) +
              "]=" + std::to_string(vis_count[e]) + " outside 1.." + std::to_string(length[x]));
  }
  // token offsets are the preorder prefix sums (_preorder_offsets, forest.py:148-157)
  {
    std::vector<int64_t> off(N, 0);
    int64_t pos = 0, pops = 0;
    std::vector<int64_t> stack{0};
    bool runaway = false;
    while (N > 0 && !stack.empty()) {
      const int64_t x = stack.back();
      stack.pop_back();
      if (++pops > 4 * N + 4) {  // a cyclic children list: offsets cannot match
        runaway = true;
        break;
      }
      off[x] = pos;
      pos += length[x];
      for (int64_t j = children_ptr[x + 1] - 1; j >= children_ptr[x]; --j) stack.push_back(children_idx[j]);
    }
    bool same = !runaway && n_token_offset == N && std::equal(off.begin(), off.end(), token_offset);
    if (!same) add(CODEC_VIOLATION_FLATTEN_MISMATCH, kNone, kNone, "token offsets are not the preorder prefix sums");
  }
  *out = rep;
  return CODEC_OK;
}

extern "C" int32_t codec_report_count(const codec_report* rep, int64_t* n) {
  if (!rep || !n) return fail(CODEC_ERR_VALUE, "NULL argument");
  *n = (int64_t)rep->recs.size();
  return CODEC_OK;
}

extern "C" int32_t codec_report_get(const codec_report* rep, int64_t i, int32_t* code, int64_t* node,
                                    int64_t* request, char* msg, int64_t msg_cap) {
  if (!rep || i < 0 || i >= (int64_t)rep->recs.size()) return fail(CODEC_ERR_VALUE, "no violation %lld", (long long)i);
  const Rec& r = rep->recs[i];
  if (code) *code = r.code;
  if (node) *node = r.node;
  if (request) *request = r.request;
  if (msg && msg_cap > 0) {
    const int64_t n = std::min<int64_t>(msg_cap - 1, (int64_t)r.msg.size());
    std::copy(r.msg.begin(), r.msg.begin() + n, msg);
    msg[n] = '\0';
  }
  return CODEC_OK;
}

extern "C" void codec_report_free(codec_report* rep) { delete rep; }

// ------------------------------------------------------------ cost profiles
// Rows (n_q, n, cost) in file order -> knots (sorted unique) and the
// n-major grid. The first offending row decides the error, duplicate
// before cost within a row; then the first missing cell in n-major order.
extern "C" int32_t codec_cost_grid(int64_t n_rows, const int64_t* row_nq, const int64_t* row_n, const double* row_cost,
                                   int32_t* n_nq, int32_t* n_n, int64_t* nq_knots, int64_t* n_knots, double* grid) {
  if (n_rows < 0 || !n_nq || !n_n) return fail(CODEC_ERR_VALUE, "NULL argument");
  std::map<std::pair<int64_t, int64_t>, double> cells;  // (n, n_q) -> cost
  std::set<int64_t> kq, kn;
  for (int64_t i = 0; i < n_rows; ++i) {
    kq.insert(row_nq[i]);
    kn.insert(row_n[i]);
    const auto key = std::make_pair(row_n[i], row_nq[i]);
    if (!cells.emplace(key, row_cost[i]).second)
      return fail(CODEC_ERR_DUPLICATE_KNOT, "cell (n_q=%lld, n=%lld) appears twice", (long long)row_nq[i],
                  (long long)row_n[i]);
    if (!(row_cost[i] > 0))
      return fail(CODEC_ERR_NON_POSITIVE_COST, "cell (n_q=%lld, n=%lld) has non-positive cost %s",
                  (long long)row_nq[i], (long long)row_n[i], py_float(row_cost[i]).c_str());
  }
  *n_nq = (int32_t)kq.size();
  *n_n = (int32_t)kn.size();
  if (!grid) return CODEC_OK;  // sizing call
  int32_t j = 0;
  for (int64_t x : kq) nq_knots[j++] = x;
  j = 0;
  for (int64_t x : kn) n_knots[j++] = x;
  int64_t at = 0;
  for (int64_t n : kn)
    for (int64_t q : kq) {
      auto it = cells.find({n, q});
      if (it == cells.end())
        return fail(CODEC_ERR_INCOMPLETE_GRID, "grid is missing cell (n_q=%lld, n=%lld)", (long long)q, (long long)n);
      grid[at++] = it->second;
    }
  return CODEC_OK;
}

extern "C" int32_t codec_cost_table_check(int32_t n_nq, const int64_t* nq_knots, int32_t n_n, const int64_t* n_knots,
                                          int32_t grid_ndim, const int64_t* grid_shape, const double* cost_ms) {
  if ((n_nq && !nq_knots) || (n_n && !n_knots) || !grid_shape) return fail(CODEC_ERR_VALUE, "NULL argument");
  if (!(grid_ndim == 2 && grid_shape[0] == n_n && grid_shape[1] == n_nq))
    return fail(CODEC_ERR_INCOMPLETE_GRID, "grid %s does not match knots (%d, %d)",
                py_tuple(grid_shape, grid_ndim).c_str(), n_n, n_nq);
  struct K {
    const char* name;
    const int64_t* k;
    int32_t n;
  };
  for (const K& kk : {K{"n_q", nq_knots, n_nq}, K{"n", n_knots, n_n}})
    for (int32_t i = 0; i < kk.n; ++i)
      if (kk.k[i] < 1 || (i && kk.k[i] <= kk.k[i - 1]))
        return fail(CODEC_ERR_DUPLICATE_KNOT, "%s knots must be strictly ascending positives: %s", kk.name,
                    py_tuple(kk.k, kk.n).c_str());
  for (int64_t i = 0; i < (int64_t)n_n * n_nq; ++i)
    if (!(cost_ms[i] > 0)) return fail(CODEC_ERR_NON_POSITIVE_COST, "every grid cost must be > 0");
  return CODEC_OK;
}
