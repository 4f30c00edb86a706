// K0: forest indexing on the host (C++), exported through the C ABI.
//
// Restates the structural half of build_forest() (reference
// forest.py:160-251): node/parent validation (:186-206), request path
// validation (:218-234), ascending query sets I_n (:236-237),
// visible_len validation (:238-247) and the preorder token offsets kappa
// (_preorder_offsets, :148-157). Messages match the reference's so the
// Python layer can raise the same exception text.
#include <algorithm>
#include <unordered_map>
#include <vector>

#include "common.h"

struct codec_index {
  int32_t n_nodes = 0, bs = 0;
  std::vector<int64_t> length, node_off;
  std::vector<int64_t> qset_ptr, qset_vis, child_ptr;
  std::vector<int32_t> qset_idx, child_idx;
  std::vector<int64_t> path_ptr;
  std::vector<int32_t> path_idx;
  int64_t total_tokens = 0, path_nnz = 0;
};

namespace codec {
std::string& last_error() {
  thread_local std::string msg;
  return msg;
}
}  // namespace codec

using codec::fail;

extern "C" const char* codec_last_error(void) { return codec::last_error().c_str(); }
extern "C" int32_t codec_abi_version(void) { return 8; }

extern "C" int32_t codec_index_build(int32_t n_nodes, const int32_t* parent, const int64_t* length,
                                     int32_t bs, const int64_t* path_ptr, const int32_t* path_idx,
                                     int64_t n_vis, const int32_t* vis_node, const int32_t* vis_req,
                                     const int64_t* vis_count, codec_index** out) {
  if (!out) return fail(CODEC_ERR_VALUE, "out handle is NULL");
  *out = nullptr;
  if (n_nodes < 2) return fail(CODEC_ERR_DIMENSION_MISMATCH, "forest needs at least one node");
  auto ix = new codec_index();
  ix->n_nodes = n_nodes;
  ix->bs = bs;
  ix->length.assign(length, length + n_nodes);
  ix->length[0] = 0;

  // nodes: ids 1..N in declaration order, parent already declared
  for (int32_t nid = 1; nid < n_nodes; ++nid) {
    int32_t p = parent[nid];
    if (p == nid) {
      delete ix;
      return fail(CODEC_ERR_CYCLE_DETECTED, "node %d is its own parent", nid);
    }
    if (p < 0 || p >= nid) {
      delete ix;
      return fail(CODEC_ERR_DANGLING_PARENT, "node %d references undeclared parent %d", nid, p);
    }
    if (ix->length[nid] < 1) {
      delete ix;
      return fail(CODEC_ERR_DIMENSION_MISMATCH, "node %d has no tokens", nid);
    }
  }

  // children CSR in declaration order
  std::vector<int64_t> nkids(n_nodes, 0);
  for (int32_t nid = 1; nid < n_nodes; ++nid) nkids[parent[nid]]++;
  ix->child_ptr.assign(n_nodes + 1, 0);
  for (int32_t i = 0; i < n_nodes; ++i) ix->child_ptr[i + 1] = ix->child_ptr[i] + nkids[i];
  ix->child_idx.assign(n_nodes - 1, 0);
  {
    std::vector<int64_t> fill(ix->child_ptr.begin(), ix->child_ptr.end() - 1);
    for (int32_t nid = 1; nid < n_nodes; ++nid) ix->child_idx[fill[parent[nid]]++] = nid;
  }

  // request paths: parent -> child chains starting under the virtual root
  std::vector<int64_t> qcount(n_nodes, 0);
  for (int32_t r = 0; r < bs; ++r) {
    int64_t a = path_ptr[r], b = path_ptr[r + 1];
    if (a == b) {
      delete ix;
      return fail(CODEC_ERR_PATH_NOT_PREFIX_CHAIN, "request %d has an empty path", r);
    }
    int32_t prev = 0;
    for (int64_t i = a; i < b; ++i) {
      int32_t nid = path_idx[i];
      if (nid < 1 || nid >= n_nodes) {
        delete ix;
        return fail(CODEC_ERR_PATH_NOT_PREFIX_CHAIN, "request %d path references missing node %d", r, nid);
      }
      if (parent[nid] != prev) {
        delete ix;
        return fail(CODEC_ERR_PATH_NOT_PREFIX_CHAIN, "request %d: %d->%d is not a parent->child edge",
                    r, prev, nid);
      }
      qcount[nid]++;
      prev = nid;
    }
  }
  ix->path_nnz = path_ptr[bs] - path_ptr[0];
  ix->path_ptr.assign(bs + 1, 0);
  for (int32_t r = 0; r <= bs; ++r) ix->path_ptr[r] = path_ptr[r] - path_ptr[0];
  ix->path_idx.assign(path_idx + path_ptr[0], path_idx + path_ptr[bs]);

  // query sets: iterating requests in ascending order keeps each I_n sorted
  ix->qset_ptr.assign(n_nodes + 1, 0);
  for (int32_t i = 0; i < n_nodes; ++i) ix->qset_ptr[i + 1] = ix->qset_ptr[i] + qcount[i];
  ix->qset_idx.assign(ix->qset_ptr[n_nodes], 0);
  ix->qset_vis.assign(ix->qset_ptr[n_nodes], 0);
  {
    std::vector<int64_t> fill(ix->qset_ptr.begin(), ix->qset_ptr.end() - 1);
    for (int32_t r = 0; r < bs; ++r)
      for (int64_t i = path_ptr[r]; i < path_ptr[r + 1]; ++i) {
        int32_t nid = path_idx[i];
        int64_t pos = fill[nid]++;
        ix->qset_idx[pos] = r;
        ix->qset_vis[pos] = ix->length[nid];
      }
  }

  // visible_len: request must be routed through the node, count in 1..len
  for (int64_t e = 0; e < n_vis; ++e) {
    int32_t nid = vis_node[e], r = vis_req[e];
    int64_t cnt = vis_count[e];
    if (nid < 1 || nid >= n_nodes) {
      delete ix;
      return fail(CODEC_ERR_UNKNOWN_NODE, "no node %d", nid);
    }
    const int32_t* lo = ix->qset_idx.data() + ix->qset_ptr[nid];
    const int32_t* hi = ix->qset_idx.data() + ix->qset_ptr[nid + 1];
    const int32_t* it = std::lower_bound(lo, hi, r);
    if (it == hi || *it != r) {
      delete ix;
      return fail(CODEC_ERR_PATH_NOT_PREFIX_CHAIN,
                  "visible_len on node %d names request %d not routed through it", nid, r);
    }
    if (cnt < 1 || cnt > ix->length[nid]) {
      const long long nl = (long long)ix->length[nid];
      delete ix;
      return fail(CODEC_ERR_DIMENSION_MISMATCH, "node %d: visible_len[%d]=%lld outside 1..%lld", nid, r,
                  (long long)cnt, nl);
    }
    ix->qset_vis[it - ix->qset_idx.data()] = cnt;
  }

  // preorder flattening: explicit stack, first-declared child popped first
  ix->node_off.assign(n_nodes, 0);
  {
    std::vector<int32_t> stack;
    stack.reserve(n_nodes);
    stack.push_back(0);
    int64_t cursor = 0;
    while (!stack.empty()) {
      int32_t nid = stack.back();
      stack.pop_back();
      ix->node_off[nid] = cursor;
      cursor += ix->length[nid];
      for (int64_t c = ix->child_ptr[nid + 1] - 1; c >= ix->child_ptr[nid]; --c)
        stack.push_back(ix->child_idx[c]);
    }
    ix->total_tokens = cursor;
  }
  *out = ix;
  return CODEC_OK;
}

extern "C" void codec_index_free(codec_index* ix) { delete ix; }

extern "C" int32_t codec_index_info_get(const codec_index* ix, codec_index_info* info) {
  if (!ix || !info) return fail(CODEC_ERR_VALUE, "NULL argument");
  info->n_nodes = ix->n_nodes;
  info->bs = ix->bs;
  info->total_tokens = ix->total_tokens;
  info->qset_nnz = (int64_t)ix->qset_idx.size();
  info->path_nnz = ix->path_nnz;
  return CODEC_OK;
}

extern "C" int32_t codec_index_read(const codec_index* ix, int64_t* node_off, int64_t* qset_ptr,
                                    int32_t* qset_idx, int64_t* qset_vis, int64_t* children_ptr,
                                    int32_t* children_idx) {
  if (!ix) return fail(CODEC_ERR_VALUE, "NULL index");
  if (node_off) std::copy(ix->node_off.begin(), ix->node_off.end(), node_off);
  if (qset_ptr) std::copy(ix->qset_ptr.begin(), ix->qset_ptr.end(), qset_ptr);
  if (qset_idx) std::copy(ix->qset_idx.begin(), ix->qset_idx.end(), qset_idx);
  if (qset_vis) std::copy(ix->qset_vis.begin(), ix->qset_vis.end(), qset_vis);
  if (children_ptr) std::copy(ix->child_ptr.begin(), ix->child_ptr.end(), children_ptr);
  if (children_idx) std::copy(ix->child_idx.begin(), ix->child_idx.end(), children_idx);
  return CODEC_OK;
}

// Internal accessors for host_table.cpp
namespace codec {
const std::vector<int64_t>& ix_node_off(const codec_index* ix) { return ix->node_off; }
const std::vector<int64_t>& ix_length(const codec_index* ix) { return ix->length; }
const std::vector<int64_t>& ix_qset_ptr(const codec_index* ix) { return ix->qset_ptr; }
const std::vector<int32_t>& ix_qset_idx(const codec_index* ix) { return ix->qset_idx; }
const std::vector<int64_t>& ix_qset_vis(const codec_index* ix) { return ix->qset_vis; }
const std::vector<int64_t>& ix_path_ptr(const codec_index* ix) { return ix->path_ptr; }
const std::vector<int32_t>& ix_path_idx(const codec_index* ix) { return ix->path_idx; }
int32_t ix_bs(const codec_index* ix) { return ix->bs; }
int32_t ix_n_nodes(const codec_index* ix) { return ix->n_nodes; }
int64_t ix_total_tokens(const codec_index* ix) { return ix->total_tokens; }
}  // namespace codec
