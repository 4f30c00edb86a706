// Device task table: a DivisionPlan expanded into GPU work groups.
//
// Host C++ restatement of the job construction of the reference
// executor: plan/forest agreement (_plan_slices, executor.py:120-142),
// per-subtask row filter `visible_count(r) > start` (:156), per-row
// visible clip `min(visible, stop) - start` (:187-190), and each
// request's partial list in path-then-slice order (_reduce_one,
// executor.py:211-224). The result is one int32 blob (uploaded once and
// reused across decode steps) plus counts/offsets (codec_table_info).
//
// Group = (subtask, row tile). A row tile is up to 128/g requests for the
// tcgen05 kernel (one M=128 tile of query-head rows) or one request for
// the GEMV / generic kernels. CTA = group x local kv head.
#include <algorithm>
#include <array>
#include <cstdlib>
#include <map>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "common.h"
#include "device_table.h"

using codec::fail;
using codec::fail_str;

namespace codec {
const std::vector<int64_t>& ix_node_off(const codec_index* ix);
const std::vector<int64_t>& ix_length(const codec_index* ix);
const std::vector<int64_t>& ix_qset_ptr(const codec_index* ix);
const std::vector<int32_t>& ix_qset_idx(const codec_index* ix);
const std::vector<int64_t>& ix_qset_vis(const codec_index* ix);
const std::vector<int64_t>& ix_path_ptr(const codec_index* ix);
const std::vector<int32_t>& ix_path_idx(const codec_index* ix);
int32_t ix_bs(const codec_index* ix);
int32_t ix_n_nodes(const codec_index* ix);
int64_t ix_total_tokens(const codec_index* ix);
}  // namespace codec

struct codec_table {
  codec_table_info info{};
  std::vector<int32_t> blob;
};

namespace {
// Most query-head rows a slice may have to take the multi-request kernel
// (CODEC_MULTI_MAX_ROWS overrides kMultiMaxRows; tuning, must match
// scheduler.MULTI_MAX_ROWS)
int64_t multi_max_rows() {
  static const int64_t v = [] {
    const char* e = getenv("CODEC_MULTI_MAX_ROWS");
    return e ? (int64_t)atoll(e) : (int64_t)codec::kMultiMaxRows;
  }();
  return v;
}
// ... and the transposed tensor-core kernel (CODEC_TCT_MAX_ROWS overrides
// kTctMaxRows; must match scheduler.TCT_MAX_ROWS)
int64_t tct_max_rows() {
  static const int64_t v = [] {
    const char* e = getenv("CODEC_TCT_MAX_ROWS");
    return e ? (int64_t)atoll(e) : (int64_t)codec::kTctMaxRows;
  }();
  return v;
}
// CODEC_TCT_CTAS: the transposed kernel's grid (0: by KV bytes, below)
int64_t tct_ctas_env() {
  static const int64_t v = [] {
    const char* e = getenv("CODEC_TCT_CTAS");
    return e ? (int64_t)atoll(e) : (int64_t)0;
  }();
  return v;
}
// Cost of a unit boundary inside a CTA pair, in KV tiles (device balancer
// below). CODEC_TC_UNIT_COST overrides it (tuning).
int64_t tc_unit_cost() {
  static const int64_t v = [] {
    const char* e = getenv("CODEC_TC_UNIT_COST");
    return e ? (int64_t)atoll(e) : (int64_t)codec::kTcUnitCostDefault;
  }();
  return v;
}


std::string py_list(const std::vector<int64_t>& v) {
  std::ostringstream os;
  os << "[";
  for (size_t i = 0; i < v.size(); ++i) os << (i ? ", " : "") << v[i];
  os << "]";
  return os.str();
}

std::string py_ranges(const std::vector<std::pair<int64_t, int64_t>>& v) {
  std::ostringstream os;
  os << "[";
  for (size_t i = 0; i < v.size(); ++i) os << (i ? ", " : "") << "(" << v[i].first << ", " << v[i].second << ")";
  os << "]";
  return os.str();
}

bool is_pow2(int x) { return x > 0 && (x & (x - 1)) == 0; }

}  // namespace

extern "C" int32_t codec_table_build(const codec_index* ix, const codec_dims* dims, int32_t n_tasks,
                                     const int64_t* task_node, const int64_t* task_nq, int32_t n_sub,
                                     const int32_t* sub_task, const int64_t* sub_start,
                                     const int64_t* sub_stop, const int32_t* sub_block, codec_table** out) {
  using namespace codec;
  if (!ix || !dims || !out) return fail(CODEC_ERR_VALUE, "NULL argument");
  *out = nullptr;
  const int32_t n_nodes = ix_n_nodes(ix), bs = ix_bs(ix);
  const auto& len = ix_length(ix);
  const auto& qptr = ix_qset_ptr(ix);
  const auto& qidx = ix_qset_idx(ix);
  const auto& qvis = ix_qset_vis(ix);
  const auto& pptr = ix_path_ptr(ix);
  const auto& pidx = ix_path_idx(ix);
  if (dims->bs != bs) return fail(CODEC_ERR_DIMENSION_MISMATCH, "%d queries for %d requests", dims->bs, bs);
  if (dims->h_kv < 1 || dims->h_q % dims->h_kv != 0)
    return fail(CODEC_ERR_DIMENSION_MISMATCH, "h_q=%d must be a positive multiple of h_kv=%d", dims->h_q, dims->h_kv);
  if (dims->head_begin < 0 || dims->head_end > dims->h_kv || dims->head_begin >= dims->head_end)
    return fail(CODEC_ERR_VALUE, "kv head shard [%d, %d) outside 0..%d", dims->head_begin, dims->head_end, dims->h_kv);
  // paged pool: node n's token x is logical token base[n] * P + x, which
  // the kernels map through page_table to a physical pool row
  const int32_t page = dims->page_size;
  std::vector<int64_t> off_paged;
  if (page) {
    if (page < 128 || !is_pow2(page))
      return fail(CODEC_ERR_VALUE, "page_size %d must be a power of two >= 128", page);
    if (!dims->page_table) return fail(CODEC_ERR_VALUE, "page_size %d without a page table", page);
    if (dims->kv_dtype != CODEC_BF16 || dims->d != 128 || dims->h_q > 8 * dims->h_kv ||
        (dims->flags & (CODEC_FLAG_NO_TC | CODEC_FLAG_NO_GEMV | CODEC_FLAG_GEMV_SIMT)))
      return fail(CODEC_ERR_UNSUPPORTED,
                  "paged KV runs on the tensor-core and mma.sync suffix kernels only: bf16, d = 128, <= 8 "
                  "query heads per kv head");
    if (dims->pool_tokens < page) return fail(CODEC_ERR_VALUE, "paged pool of %lld tokens holds no page",
                                              (long long)dims->pool_tokens);
    off_paged.resize(n_nodes + 1, 0);
    for (int32_t n = 0; n < n_nodes; ++n) off_paged[n + 1] = off_paged[n] + (len[n] + page - 1) / page;
    if (off_paged[n_nodes] * page >= (int64_t(1) << 31))
      return fail(CODEC_ERR_UNSUPPORTED, "paged pool larger than 2^31 logical tokens");
    for (auto& x : off_paged) x *= page;
  } else if (dims->pool_tokens < ix_total_tokens(ix)) {
    return fail(CODEC_ERR_VALUE, "pool holds %lld tokens, forest needs %lld", (long long)dims->pool_tokens,
                (long long)ix_total_tokens(ix));
  }
  const auto& off = page ? off_paged : ix_node_off(ix);
  if (dims->pool_tokens >= (int64_t(1) << 31)) return fail(CODEC_ERR_UNSUPPORTED, "pool larger than 2^31 tokens");
  const int32_t g = dims->h_q / dims->h_kv;
  const int32_t d = dims->d;
  for (int32_t j = 0; j < n_tasks; ++j)
    if (task_node[j] < 1 || task_node[j] >= n_nodes)
      return fail(CODEC_ERR_PLAN_FOREST_MISMATCH, "plan task %d names node %lld outside the forest", j,
                  (long long)task_node[j]);
  for (int32_t s = 0; s < n_sub; ++s)
    if (sub_task[s] < 0 || sub_task[s] >= n_tasks)
      return fail(CODEC_ERR_PLAN_FOREST_MISMATCH, "subtask %d names task %d of %d", s, sub_task[s], n_tasks);

  // ---- plan <-> forest agreement (executor.py:120-142)
  std::set<int64_t> have, want;
  for (int32_t s = 0; s < n_sub; ++s) have.insert(task_node[sub_task[s]]);
  for (int32_t n = 1; n < n_nodes; ++n)
    if (qptr[n + 1] > qptr[n]) want.insert(n);
  if (have != want)
    return fail_str(CODEC_ERR_PLAN_FOREST_MISMATCH,
                    "plan covers nodes " + py_list({have.begin(), have.end()}) + ", forest needs " +
                        py_list({want.begin(), want.end()}));
  {
    std::vector<std::vector<std::pair<int64_t, int64_t>>> per_task(n_tasks);
    for (int32_t s = 0; s < n_sub; ++s) per_task[sub_task[s]].push_back({sub_start[s], sub_stop[s]});
    for (int32_t j = 0; j < n_tasks; ++j) {
      auto& r = per_task[j];
      std::sort(r.begin(), r.end());
      int64_t pos = 0, nl = len[task_node[j]];
      bool ok = !r.empty();
      for (auto& p : r) {
        if (p.first != pos || p.second <= p.first) ok = false;
        pos = p.second;
      }
      if (pos != nl) ok = false;
      if (!ok)
        return fail_str(CODEC_ERR_PLAN_FOREST_MISMATCH, "node " + std::to_string(task_node[j]) + " slices " +
                                                            py_ranges(r) + " do not tile 0.." + std::to_string(nl));
    }
  }
  // ---- task -> query-set chunk: tasks of a node split I_n in order
  std::vector<int64_t> chunk_lo(n_tasks), chunk_hi(n_tasks);
  {
    std::map<int64_t, std::vector<int32_t>> by_node;
    for (int32_t j = 0; j < n_tasks; ++j) by_node[task_node[j]].push_back(j);
    for (auto& kv : by_node) {
      int64_t n = kv.first, size = qptr[n + 1] - qptr[n], tot = 0;
      for (int32_t j : kv.second) tot += task_nq[j];
      int64_t hm = size > 0 ? tot / size : 0;
      bool ok = size > 0 && hm >= 1 && hm * size == tot;
      int64_t cur = 0;
      for (int32_t j : kv.second) {
        if (!ok || task_nq[j] % hm != 0) {
          ok = false;
          break;
        }
        chunk_lo[j] = cur;
        cur += task_nq[j] / hm;
        chunk_hi[j] = cur;
      }
      if (!ok || cur != size)
        return fail(CODEC_ERR_PLAN_FOREST_MISMATCH, "tasks of node %lld do not partition its query set",
                    (long long)n);
    }
  }

  // ---- kernel eligibility
  const bool tc_ok = dims->kv_dtype == CODEC_BF16 && d == 128 && is_pow2(g) && g <= 128 &&
                     !(dims->flags & CODEC_FLAG_NO_TC);
  // (the GEMV kernels are instantiated for 4 and 8 query-head rows; more
  // query heads per kv head take the generic kernel)
  const bool gemv_ok = (dims->kv_dtype == CODEC_BF16 || dims->kv_dtype == CODEC_F32) &&
                       (d == 64 || d == 128 || d == 256) && g <= 8 && !(dims->flags & CODEC_FLAG_NO_GEMV);
  const int32_t tc_reqs = tc_ok ? std::max(1, kTcGroupRows / g) : 0;
  const int32_t gemv_rows = g <= 4 ? 4 : 8;
  // lightly shared slices (2+ requests, <= kMultiMaxRows query-head rows):
  // the multi-request mma.sync kernel streams them once for all requests
  const bool multi_ok = dims->kv_dtype == CODEC_BF16 && d == 128 && g <= 8 &&
                        !(dims->flags & (CODEC_FLAG_NO_MULTI | CODEC_FLAG_GEMV_SIMT | CODEC_FLAG_NO_GEMV));
  const int32_t multi_reqs = std::max(1, kMultiRows / g);
  // slices of 2+ requests of nodes with at most tct_max_rows() query-head
  // rows in all: the transposed tensor-core kernel (work proportional to the
  // rows; one CTA per SM streams ~2x what three multi-request CTAs do), in
  // groups of kTctRows rows. (A larger node's last row chunk stays on the
  // pair kernel, in lockstep with the node's other chunks: one HBM read of
  // its KV.) The multi-request kernel takes them without it.
  const bool tct_ok = tc_ok && g <= kTctRows && !(dims->flags & (CODEC_FLAG_NO_TCT | CODEC_FLAG_FORCE_TC));
  const int64_t tc_min_rows = multi_ok ? multi_max_rows() + 1 : kTcMinRows;
  const int32_t tct_reqs = std::max(1, kTctRows / g);

  // ---- rows and slots
  struct Grp {
    int32_t kind, kv_tok, len, row_begin, n_rows, max_vis, node;
    int64_t order_len;
    int32_t start;  // slice start within the node (DecodeStep.grow)
  };
  std::vector<Grp> groups;
  std::vector<int32_t> rows;  // 4 per row: req, vis_local, slot, fused merge entry (GEMV rows) or -1
  std::vector<char> row_gemv;  // per template row: belongs to a GEMV group
  // per request: (path position, subtask, row index)
  std::vector<std::vector<std::array<int64_t, 3>>> req_units(bs);
  std::vector<std::vector<int32_t>> node_pathpos(bs);
  auto path_pos = [&](int32_t r, int64_t n) -> int64_t {
    for (int64_t i = pptr[r]; i < pptr[r + 1]; ++i)
      if (pidx[i] == n) return i - pptr[r];
    return -1;
  };
  for (int32_t s = 0; s < n_sub; ++s) {
    int32_t j = sub_task[s];
    int64_t n = task_node[j], start = sub_start[s], stop = sub_stop[s];
    std::vector<std::pair<int32_t, int32_t>> live;  // (req, vis_local)
    for (int64_t q = qptr[n] + chunk_lo[j]; q < qptr[n] + chunk_hi[j]; ++q) {
      int64_t vis = qvis[q];
      if (vis > start) live.push_back({qidx[q], (int32_t)(std::min(vis, stop) - start)});
    }
    if (live.empty()) continue;
    int kind;
    int32_t per;
    const int64_t rows_live = (int64_t)live.size() * g, rows_node = (qptr[n + 1] - qptr[n]) * (int64_t)g;
    const int64_t tct_max = (dims->flags & CODEC_FLAG_TCT_WIDE) ? (int64_t)kTctRows : tct_max_rows();
    if (tct_ok && live.size() >= 2 && rows_node <= tct_max) {
      kind = kKindTct;
      per = tct_reqs;
    } else if (tc_ok && (rows_live >= tc_min_rows || (dims->flags & CODEC_FLAG_FORCE_TC))) {
      kind = kKindTc;
      per = tc_reqs;
    } else if (multi_ok && live.size() >= 2) {
      kind = kKindMulti;
      per = multi_reqs;
    } else if (gemv_ok) {
      kind = kKindGemv;
      per = 1;
    } else {
      kind = kKindGeneric;
      per = 1;
    }
    // paged pool: every TMA box (128-token K/V tiles, 32-token suffix
    // chunks) must sit inside one page
    const int64_t box = (kind == kKindTc || kind == kKindTct) ? 128 : 32;
    if (page && start % box != 0)
      return fail(CODEC_ERR_UNSUPPORTED, "paged KV: node %lld slice starts at token %lld, not a multiple of %d",
                  (long long)n, (long long)start, (int)box);
    for (size_t a = 0; a < live.size(); a += per) {
      size_t b = std::min(live.size(), a + per);
      int32_t max_vis = 0;
      for (size_t i = a; i < b; ++i) max_vis = std::max(max_vis, live[i].second);
      Grp gr{kind, (int32_t)(off[n] + start), (int32_t)(stop - start), (int32_t)(rows.size() / 4),
             (int32_t)(b - a), max_vis, (int32_t)n, stop - start, (int32_t)start};
      for (size_t i = a; i < b; ++i) {
        int32_t r = live[i].first;
        int64_t pp = path_pos(r, n);
        if (pp < 0)
          return fail(CODEC_ERR_INCOMPLETE_PARTIALS, "request %d not on a path through node %lld", r, (long long)n);
        // TC rows are templates: their partials come from the per-head
        // pieces cut below; the other kinds' rows serve every head
        if (kind != kKindTc) req_units[r].push_back({pp, (int64_t)s, (int64_t)(rows.size() / 4)});
        row_gemv.push_back(kind == kKindGemv);
        rows.push_back(r);
        rows.push_back(live[i].second);
        rows.push_back(-1);
        rows.push_back(-1);
      }
      groups.push_back(gr);
    }
  }
  // ---- group order: TC, GEMV, generic; longest slices first within a kind
  std::stable_sort(groups.begin(), groups.end(), [](const Grp& a, const Grp& b) {
    if (a.kind != b.kind) return a.kind < b.kind;
    return a.order_len > b.order_len;
  });
  (void)sub_block;
  const int32_t h_local = dims->head_end - dims->head_begin;

  // ---- tensor-core pieces (stream-K over CTA pairs). A unit = (TC group,
  // local kv head) of ceil(max_vis / 128) KV tiles. Units are laid out in
  // lanes -- lane c holds the c-th row chunk of every KV slice -- and each
  // lane's unit sequence (slice, head order) is cut into equal tile ranges,
  // one per CTA pair of the lane: every pair gets the same work, at most
  // a couple of pieces (few epilogues, few partials), and pair j of every
  // lane walks the same K/V tiles at the same time, so a tile is read from
  // HBM once and from L2 by the other lanes. Pieces never cross plan
  // slices; the reference plan's division stays the outer structure.
  struct Piece {
    int32_t grp, head, t0, t1, pair;
  };
  std::vector<Piece> pieces;
  const int64_t kTcUnitCost = tc_unit_cost();
  std::vector<int32_t> tcg;  // indices of TC groups in `groups`
  for (size_t i = 0; i < groups.size(); ++i)
    if (groups[i].kind == kKindTc) tcg.push_back((int32_t)i);
  int32_t n_pairs = 0;
  if (!tcg.empty()) {
    int32_t sms = dims->sm_count > 0 ? dims->sm_count : 148;
    if (dims->tc_sm_budget > 0) sms = std::min(sms, dims->tc_sm_budget);
    const int32_t pairs = std::max(1, sms / kTcCtasPerBlock);
    auto tiles_of = [&](int32_t gi) { return (int64_t)(groups[gi].max_vis + 127) / 128; };
    // lane = rank of the group among the TC groups of its KV slice
    std::map<std::pair<int32_t, int32_t>, std::vector<int32_t>> by_slice;  // (kv_tok, len) -> groups
    for (int32_t gi : tcg) by_slice[{groups[gi].kv_tok, groups[gi].len}].push_back(gi);
    // Slices with more lanes first: every lane then walks the slices it
    // shares with lane 0 as a PREFIX of lane 0's sequence, at the same
    // positions -- pair k of every lane reads the same K/V tiles at the same
    // time (one HBM read, L2 hits for the others) even when slices have
    // different lane counts (cfg4: 1..7 lanes; pool order re-read ~4 GB).
    std::vector<std::pair<std::pair<int32_t, int32_t>, std::vector<int32_t>>> slices(by_slice.begin(), by_slice.end());
    std::stable_sort(slices.begin(), slices.end(),
                     [](const auto& a, const auto& b) { return a.second.size() > b.second.size(); });
    std::vector<std::vector<int32_t>> lanes;
    for (auto& kv : slices) {
      auto v = kv.second;
      std::stable_sort(v.begin(), v.end(), [&](int32_t a, int32_t b) { return groups[a].row_begin < groups[b].row_begin; });
      for (size_t c = 0; c < v.size(); ++c) {
        if (lanes.size() <= c) lanes.emplace_back();
        lanes[c].push_back(v[c]);
      }
    }
    std::vector<int64_t> lane_w(lanes.size(), 0);
    int64_t w_all = 0;
    for (size_t c = 0; c < lanes.size(); ++c) {
      for (int32_t gi : lanes[c]) lane_w[c] += tiles_of(gi) * h_local;
      w_all += lane_w[c];
    }
    // Every pair gets a budget of C cost units, a KV tile costing 1 and
    // every piece after a pair's first kTcUnitCost more (a unit boundary
    // inside a pair costs an epilogue and a pipeline refill, ~4-5 us on
    // B200: the pairs that cross one ran ~7 % longer for the same tiles).
    // Each lane's unit sequence is cut greedily into C-unit pairs of its own
    // (in lockstep with the other lanes: the same sequence is cut the same
    // way); what does not fill a whole pair -- the ends of the lanes, which
    // cover the same KV region in every lane -- is pooled in lane order and
    // cut the same way for the remaining pairs. (Whole lanes only would
    // idle pairs whenever the lane count does not divide them: 10 of 74 at
    // 16 lanes.) C is the smallest budget that needs no more than `pairs`
    // pairs; with kTcUnitCost = 0 it is ceil(W / pairs).
    struct Cut {
      int32_t gi, h;
      int64_t t0, t1, pair;
    };
    auto cut_lane = [&](const std::vector<std::pair<int32_t, int32_t>>& units,
                        const std::vector<std::array<int64_t, 2>>& ranges, int64_t C, int64_t pair_base,
                        std::vector<Cut>* out, std::vector<std::array<int64_t, 4>>* left) {
      // greedy: returns the closed pairs; the open one's pieces go to *left
      int64_t closed = 0, cost = 0;
      size_t open_begin = out ? out->size() : 0;
      std::vector<std::array<int64_t, 4>> cur;  // (unit index, t0, t1) of the open pair
      for (size_t u = 0; u < units.size(); ++u) {
        int64_t t = ranges[u][0];
        const int64_t nt = ranges[u][1];
        while (t < nt) {
          const int64_t extra = cur.empty() ? 0 : kTcUnitCost;
          const int64_t room = C - cost - extra;
          if (room <= 0) {
            ++closed;
            cost = 0;
            cur.clear();
            if (out) open_begin = out->size();
            continue;
          }
          const int64_t take = std::min(nt - t, room);
          cur.push_back({(int64_t)u, t, t + take, 0});
          if (out) out->push_back({units[u].first, units[u].second, t, t + take, pair_base + closed});
          cost += take + extra;
          t += take;
          if (cost >= C) {
            ++closed;
            cost = 0;
            cur.clear();
            if (out) open_begin = out->size();
          }
        }
      }
      if (out) out->resize(open_begin);  // the open pair's pieces are not this lane's
      if (left)
        for (auto& x : cur) left->push_back(x);
      return closed;
    };
    // lane unit sequences: (group, head) with tile ranges [0, tiles)
    std::vector<std::vector<std::pair<int32_t, int32_t>>> lane_units(lanes.size());
    std::vector<std::vector<std::array<int64_t, 2>>> lane_ranges(lanes.size());
    for (size_t c = 0; c < lanes.size(); ++c)
      for (int32_t gi : lanes[c])
        for (int32_t h = 0; h < h_local; ++h) {
          lane_units[c].push_back({gi, h});
          lane_ranges[c].push_back({0, tiles_of(gi)});
        }
    // pairs a budget C needs (lane pairs + pooled tail pairs)
    auto pool_of = [&](int64_t C, std::vector<std::pair<int32_t, int32_t>>* pu,
                       std::vector<std::array<int64_t, 2>>* pr) {
      int64_t used_c = 0;
      for (size_t c = 0; c < lanes.size(); ++c) {
        std::vector<std::array<int64_t, 4>> left;
        used_c += cut_lane(lane_units[c], lane_ranges[c], C, 0, nullptr, &left);
        for (auto& x : left) {
          pu->push_back(lane_units[c][x[0]]);
          pr->push_back({x[1], x[2]});
        }
      }
      return used_c;
    };
    auto pairs_needed = [&](int64_t C) {
      std::vector<std::pair<int32_t, int32_t>> pu;
      std::vector<std::array<int64_t, 2>> pr;
      const int64_t used_c = pool_of(C, &pu, &pr);
      std::vector<std::array<int64_t, 4>> left;
      const int64_t tail_c = cut_lane(pu, pr, C, 0, nullptr, &left);
      return used_c + tail_c + (left.empty() ? 0 : 1);
    };
    int64_t lo = std::max<int64_t>(1, (w_all + pairs - 1) / pairs), hi = lo;
    while (pairs_needed(hi) > pairs) hi = hi * 2;
    while (lo < hi) {  // smallest budget that fits (pairs_needed is non-increasing in C)
      const int64_t mid = (lo + hi) / 2;
      if (pairs_needed(mid) <= pairs) hi = mid; else lo = mid + 1;
    }
    const int64_t C = lo;
    std::vector<Cut> cuts;
    int64_t pair0 = 0;
    std::vector<std::pair<int32_t, int32_t>> pool_u;
    std::vector<std::array<int64_t, 2>> pool_r;
    for (size_t c = 0; c < lanes.size(); ++c) {
      std::vector<std::array<int64_t, 4>> left;
      pair0 += cut_lane(lane_units[c], lane_ranges[c], C, pair0, &cuts, &left);
      for (auto& x : left) {
        pool_u.push_back(lane_units[c][x[0]]);
        pool_r.push_back({x[1], x[2]});
      }
    }
    {
      std::vector<std::array<int64_t, 4>> left;
      const int64_t tail_closed = cut_lane(pool_u, pool_r, C, pair0, &cuts, &left);
      for (auto& x : left)  // the last, partly filled tail pair
        cuts.push_back({pool_u[x[0]].first, pool_u[x[0]].second, x[1], x[2], pair0 + tail_closed});
      n_pairs = (int32_t)(pair0 + tail_closed + (left.empty() ? 0 : 1));
    }
    for (auto& x : cuts) pieces.push_back({x.gi, x.h, (int32_t)x.t0, (int32_t)x.t1, (int32_t)x.pair});
  }
  // piece rows (their own records: visible tokens within the piece) and the
  // per-(request, head) TC contributions, in piece order
  struct TcRow {
    int32_t head, row;
  };
  std::vector<std::vector<TcRow>> req_tc(bs);
  struct PieceRec {
    int32_t kv_tok, len, row_begin, n_rows, max_vis, node, pair, head;
  };
  std::vector<PieceRec> prec;
  for (auto& pc : pieces) {
    const Grp& gr = groups[pc.grp];
    const int64_t tok0 = (int64_t)pc.t0 * 128, tok1 = std::min<int64_t>((int64_t)pc.t1 * 128, gr.len);
    PieceRec rec{(int32_t)(gr.kv_tok + tok0), (int32_t)(tok1 - tok0), (int32_t)(rows.size() / 4), 0, 0, gr.node,
                 pc.pair, pc.head};
    for (int32_t k = 0; k < gr.n_rows; ++k) {
      const int32_t r = rows[4 * (gr.row_begin + k)], vis = rows[4 * (gr.row_begin + k) + 1];
      const int64_t v = std::min<int64_t>(vis, tok1) - tok0;
      if (v <= 0) continue;
      req_tc[r].push_back({pc.head, (int32_t)(rows.size() / 4)});
      rows.push_back(r);
      rows.push_back((int32_t)v);
      rows.push_back(-1);
      rows.push_back(-1);
      ++rec.n_rows;
      rec.max_vis = std::max<int32_t>(rec.max_vis, (int32_t)v);
    }
    // consecutive request ids: the kernel loads the piece's Q rows with TMA
    rec.node = rec.n_rows > 0 ? rows[4 * rec.row_begin] : -1;
    for (int32_t k = 1; k < rec.n_rows; ++k)
      if (rows[4 * (rec.row_begin + k)] != rec.node + k) rec.node = -1;
    if (rec.n_rows > 0) prec.push_back(rec);
  }
  // ---- slots. Per request and kv head: the shared (GEMV / generic) partials
  // serve every head, the TC pieces only theirs. A (request, head) with a
  // single partial writes the output directly; otherwise its partials get
  // slots base, base + 1, ... (shared first) and one merge entry. Partial
  // storage is slot * hq_local + q head, so heads never collide.
  std::vector<int32_t> merge_req, merge_ptr{0}, merge_slot;
  // entries merged by the mma.sync suffix kernel itself (its partial is the
  // request's only non-TC one; the TC pieces finished before it started):
  // kept after the others, the merge kernel runs only the others
  std::vector<int32_t> fz_req, fz_ptr{0}, fz_slot, fz_row;
  const bool mma_suffix = dims->kv_dtype == CODEC_BF16 && d == 128 && g <= 8 && !(dims->flags & CODEC_FLAG_GEMV_SIMT) &&
                          (dims->flags & CODEC_FLAG_FUSED_MERGE);
  // MERGE_ALL (the fused peer-store gather): single-partial (request,
  // head) pairs get a slot and a merge entry too, so only the merge kernel
  // writes outputs
  const bool merge_all = (dims->flags & CODEC_FLAG_MERGE_ALL) != 0;
  int32_t n_slots = 0, max_merge = 0;
  for (int32_t r = 0; r < bs; ++r) {
    auto& u = req_units[r];
    std::sort(u.begin(), u.end());  // path-then-slice order
    std::vector<int32_t> n_tc(h_local, 0);
    for (auto& e : req_tc[r]) ++n_tc[e.head];
    const int32_t ns = (int32_t)u.size();
    int32_t most = 0;
    bool any_tc = false;
    for (int32_t h = 0; h < h_local; ++h) {
      most = std::max(most, ns + n_tc[h]);
      any_tc |= n_tc[h] > 0;
    }
    if (most == 0) return fail(CODEC_ERR_NO_VISIBLE_TOKENS, "request %d has no visible tokens anywhere on its path", r);
    if (most == 1 && !merge_all) {  // one partial on every head: direct
      if (ns == 1) rows[4 * u[0][2] + 2] = -1 - r;
      for (auto& e : req_tc[r]) rows[4 * e.row + 2] = -1 - r;
      continue;
    }
    const int32_t base = n_slots;
    n_slots += most;
    for (int32_t i = 0; i < ns; ++i) rows[4 * u[i][2] + 2] = base + i;
    std::vector<int32_t> next(h_local, ns);
    for (auto& e : req_tc[r]) {
      if (ns + n_tc[e.head] == 1 && !merge_all) {
        rows[4 * e.row + 2] = -1 - r;  // this head has just this piece
      } else {
        rows[4 * e.row + 2] = base + next[e.head]++;
      }
    }
    bool all_heads = true;
    for (int32_t h = 0; h < h_local; ++h) all_heads &= n_tc[h] > 0;
    int32_t tc_most = 0;
    for (int32_t h = 0; h < h_local; ++h) tc_most = std::max(tc_most, n_tc[h]);
    const bool fused = mma_suffix && !merge_all && ns == 1 && row_gemv[u[0][2]] && all_heads && tc_most <= 8 &&
                       g * 8 <= 64;
    if (fused) fz_row.push_back((int32_t)u[0][2]);
    for (int32_t h = 0; h < h_local; ++h) {
      const int32_t tot = ns + n_tc[h];
      if (tot < (merge_all ? 1 : 2)) continue;
      max_merge = std::max(max_merge, tot);
      auto& rq = fused ? fz_req : merge_req;
      auto& pt = fused ? fz_ptr : merge_ptr;
      auto& sl = fused ? fz_slot : merge_slot;
      rq.push_back(r * h_local + h);
      for (int32_t i = 0; i < tot; ++i) sl.push_back(base + i);
      pt.push_back((int32_t)sl.size());
    }
    (void)any_tc;
  }

  // fused entries after the others; a fused GEMV row's 4th field = the
  // entry of its request's kv head 0 (heads follow contiguously)
  const int32_t n_merge_plain = (int32_t)merge_req.size();
  for (size_t i = 0; i < fz_row.size(); ++i) rows[4 * fz_row[i] + 3] = n_merge_plain + (int32_t)(i * h_local);
  merge_req.insert(merge_req.end(), fz_req.begin(), fz_req.end());
  for (size_t i = 1; i < fz_ptr.size(); ++i) merge_ptr.push_back((int32_t)merge_slot.size() + fz_ptr[i]);
  merge_slot.insert(merge_slot.end(), fz_slot.begin(), fz_slot.end());

  auto t = new codec_table();
  codec_table_info& in = t->info;
  in.h_local = h_local;
  in.max_merge = max_merge;
  // the merge kernel's all-loads-in-flight width: the smallest of 4 / 8 / 16
  // that holds 95 % of the entries (the rest take its looped path) -- its
  // registers grow with the width and cut the resident merge CTAs (cfg4:
  // 37440 entries, 98 % with <= 4 partials, the largest 31)
  {
    std::vector<int32_t> cnt_np(17, 0);
    int32_t n_e = 0;
    for (size_t i = 0; i + 1 < merge_ptr.size() && (int32_t)i < n_merge_plain; ++i, ++n_e)
      ++cnt_np[std::min(16, merge_ptr[i + 1] - merge_ptr[i])];
    in.merge_np = 16;
    const char* env = getenv("CODEC_MERGE_NP");  // (experiments)
    if (env) in.merge_np = atoi(env);
    for (int w : {4, 8}) {
      if (env) break;
      int32_t within = 0;
      for (int k = 0; k <= w; ++k) within += cnt_np[k];
      if (n_e == 0 || (int64_t)within * 100 >= (int64_t)n_e * 95) {
        in.merge_np = w;
        break;
      }
    }
  }
  in.gemv_rows = gemv_rows;
  std::vector<int32_t>& blob = t->blob;
  auto emit_groups = [&](int kind, int32_t& count, int32_t& offset) {
    offset = (int32_t)blob.size();
    count = 0;
    for (auto& gr : groups)
      if (gr.kind == kind) {
        int32_t rec[kGroupInts] = {gr.kv_tok, gr.len, gr.row_begin, gr.n_rows, gr.max_vis, gr.node, gr.start, 0};
        blob.insert(blob.end(), rec, rec + kGroupInts);
        ++count;
      }
  };
  // ---- TC pieces, grouped per pair (each pair walks its list in order)
  {
    std::stable_sort(prec.begin(), prec.end(), [](const PieceRec& a, const PieceRec& b) { return a.pair < b.pair; });
    in.off_tc = (int32_t)blob.size();
    in.n_tc_groups = (int32_t)prec.size();
    std::vector<int32_t> block_ptr(n_pairs + 1, 0);
    for (auto& pr : prec) {
      int32_t rec[kGroupInts] = {pr.kv_tok, pr.len, pr.row_begin, pr.n_rows, pr.max_vis, pr.node, pr.pair, pr.head};
      blob.insert(blob.end(), rec, rec + kGroupInts);
      ++block_ptr[pr.pair + 1];
    }
    for (int32_t b = 0; b < n_pairs; ++b) block_ptr[b + 1] += block_ptr[b];
    in.n_tc_blocks = prec.empty() ? 0 : n_pairs;
    in.off_tc_block_ptr = (int32_t)blob.size();
    blob.insert(blob.end(), block_ptr.begin(), block_ptr.end());
  }
  emit_groups(kKindGemv, in.n_gemv_groups, in.off_gemv);
  emit_groups(kKindGeneric, in.n_gen_groups, in.off_gen);
  emit_groups(kKindMulti, in.n_multi_groups, in.off_multi);
  // right after the multi-request records: groups of <= 64 rows (the
  // narrow kernel) first, then those of 65..128 rows (the wide one)
  {
    in.n_tct_groups = 0;
    in.n_tct_wide = 0;
    for (int wide = 0; wide < 2; ++wide)
      for (auto& gr : groups)
        if (gr.kind == kKindTct && ((int64_t)gr.n_rows * g > 64) == (wide == 1)) {
          int32_t rec[kGroupInts] = {gr.kv_tok, gr.len, gr.row_begin, gr.n_rows, gr.max_vis, gr.node, gr.start, 0};
          blob.insert(blob.end(), rec, rec + kGroupInts);
          ++in.n_tct_groups;
          in.n_tct_wide += wide;
        }
  }
  // The transposed kernel's grid: one CTA per (slice group, kv head) item by
  // default. (A programmatically dependent grid launches only once every
  // CTA of the one before it has started, so a multi-wave K2t grid holds the
  // suffix kernel back -- 1.2 ms on cfg4 -- but a one-wave persistent grid
  // sized by KV bytes was slower still: one K2t CTA per SM streams only
  // ~30-50 GB/s, cfg4 4.99 vs 3.94 ms, cfg3 158 vs 84 us. CODEC_TCT_CTAS caps
  // the grid for experiments; the kernel loops over items either way.)
  if (in.n_tct_groups) {
    const int64_t items = (int64_t)in.n_tct_groups * h_local;
    in.tct_ctas = (int32_t)(tct_ctas_env() > 0 ? std::min(items, tct_ctas_env()) : items);
  }
  in.off_rows = (int32_t)blob.size();
  in.n_rows = (int32_t)(rows.size() / 4);
  blob.insert(blob.end(), rows.begin(), rows.end());
  in.n_merge = n_merge_plain;
  in.n_merge_fused = (int32_t)fz_req.size();
  in.off_merge_req = (int32_t)blob.size();
  blob.insert(blob.end(), merge_req.begin(), merge_req.end());
  in.off_merge_ptr = (int32_t)blob.size();
  blob.insert(blob.end(), merge_ptr.begin(), merge_ptr.end());
  in.off_merge_slot = (int32_t)blob.size();
  blob.insert(blob.end(), merge_slot.begin(), merge_slot.end());
  // (request, local kv head) -> merge entry (-1: the head's only partial is
  // written straight to the output): partial producers count themselves in
  // per-entry counters the merge waits on
  {
    std::vector<int32_t> entry_of((size_t)bs * h_local, -1);
    for (size_t e = 0; e < merge_req.size(); ++e) entry_of[merge_req[e]] = (int32_t)e;
    in.off_entry_of = (int32_t)blob.size();
    blob.insert(blob.end(), entry_of.begin(), entry_of.end());
  }
  while (blob.size() % 4) blob.push_back(0);
  in.blob_len = (int64_t)blob.size();
  in.n_slots = n_slots;
  const int64_t elem = dims->kv_dtype == CODEC_F64 ? 8 : 4;
  const int64_t hq_local = (int64_t)in.h_local * g;
  int64_t o_bytes = (int64_t)n_slots * hq_local * d * elem;
  o_bytes = (o_bytes + 255) / 256 * 256;
  // partial outputs, partial (m, l), then 256 reserved bytes
  int64_t ml_bytes = ((int64_t)n_slots * hq_local * 2 * elem + 255) / 256 * 256;
  // partial outputs, partial (m, l), a 256-byte block (TC completion
  // counter), then one int32 readiness counter per merge entry
  const int64_t cnt_bytes = ((int64_t)merge_req.size() * 4 + 255) / 256 * 256;
  in.workspace_bytes = o_bytes + ml_bytes + 256 + cnt_bytes;
  *out = t;
  return CODEC_OK;
}

extern "C" void codec_table_free(codec_table* t) { delete t; }

extern "C" int32_t codec_table_info_get(const codec_table* t, codec_table_info* info) {
  if (!t || !info) return codec::fail(CODEC_ERR_VALUE, "NULL argument");
  *info = t->info;
  return CODEC_OK;
}

extern "C" int32_t codec_table_copy(const codec_table* t, int32_t* blob) {
  if (!t || !blob) return codec::fail(CODEC_ERR_VALUE, "NULL argument");
  std::copy(t->blob.begin(), t->blob.end(), blob);
  return CODEC_OK;
}

extern "C" int32_t codec_page_layout(const codec_index* ix, int32_t page_size, int64_t* node_page_base,
                                     int64_t* n_pages) {
  using namespace codec;
  if (!ix || !node_page_base || !n_pages) return fail(CODEC_ERR_VALUE, "NULL argument");
  if (page_size < 1) return fail(CODEC_ERR_VALUE, "page_size %d must be positive", page_size);
  const auto& len = ix_length(ix);
  const int32_t n_nodes = ix_n_nodes(ix);
  node_page_base[0] = 0;
  for (int32_t n = 0; n < n_nodes; ++n) node_page_base[n + 1] = node_page_base[n] + (len[n] + page_size - 1) / page_size;
  *n_pages = node_page_base[n_nodes];
  return CODEC_OK;
}
