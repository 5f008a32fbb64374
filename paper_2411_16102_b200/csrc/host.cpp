// host.cpp — descriptor builder, subtree sharder and work planner of libblend.
//
// Implements the host side of include/blend.h:
//   blend_tree_build  radix trie (PAPER §4.1, §5 P:6 "Trie Tree"), exact
//                     128-bit density keys from the cost model (§2.3 P:87-96,
//                     §4.2), layer-wise sort (Alg. 1, §4.3),
//                     preorder ids, pages, SMALL/BIG + SEPARATE/FOLD classes
//                     (§7.2) and the device work plan;
//   blend_shard       2G-block fold of the DFS request order (§7.1);
//   blend_tree_dump   golden text dump (SPEC S:238 style).
// No floating point anywhere in the descriptor path: the keys are integers and
// are compared by exact 256-bit cross products, so results are bit-identical to
// the Python-int oracle (oracle/tree.py), which shares no code with this file.
#include <algorithm>
#include <climits>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <unordered_map>
#include <vector>

#include "blend.h"
#include "internal.h"
#include "tree.h"

#ifndef BLEND_STREAM_SM_GBS
#define BLEND_STREAM_SM_GBS 68.0   // planning constant: streaming pass GB/s per SM on a partial grid
#endif

namespace {

thread_local std::string g_err;

int fail(int status, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return status;
}

std::string u128_str(u128 v) {
  if (v == 0) return "0";
  char buf[64];
  int n = 0;
  while (v) {
    buf[n++] = char('0' + int(v % 10));
    v /= 10;
  }
  std::string s(buf, buf + n);
  std::reverse(s.begin(), s.end());
  return s;
}

// a*b as a 256-bit (hi, lo) pair
struct U256 {
  u128 hi, lo;
};
U256 mul_full(u128 a, u128 b) {
  const u128 M = ~(u128)0 >> 64;
  u128 a0 = a & M, a1 = a >> 64, b0 = b & M, b1 = b >> 64;
  u128 p00 = a0 * b0, p01 = a0 * b1, p10 = a1 * b0, p11 = a1 * b1;
  u128 mid = (p00 >> 64) + (p01 & M) + (p10 & M);
  U256 r;
  r.lo = (p00 & M) | (mid << 64);
  r.hi = p11 + (p01 >> 64) + (p10 >> 64) + (mid >> 64);
  return r;
}
bool gt256(U256 a, U256 b) { return a.hi != b.hi ? a.hi > b.hi : a.lo > b.lo; }

}  // namespace


namespace {

struct TNode {
  int32_t start, len, ref, parent;
};

inline uint64_t ckey(int32_t parent, int32_t tok) {
  return (uint64_t(uint32_t(parent + 1)) << 32) | uint32_t(tok);
}

int validate(const blend_build_args* a) {
  if (!a) return fail(BLEND_EINVAL, "args is NULL");
  if (a->num_q_heads <= 0 || a->num_kv_heads <= 0 || a->num_q_heads % a->num_kv_heads != 0)
    return fail(BLEND_EINVAL, "num_q_heads must be a positive multiple of num_kv_heads");
  if (a->head_dim != 64 && a->head_dim != 128) return fail(BLEND_EUNSUPPORTED, "head_dim must be 64 or 128");
  int ps = a->page_size;
  if (ps < 16 || ps > 128 || (ps & (ps - 1)) != 0)
    return fail(BLEND_EINVAL, "page_size must be a power of two in [16,128]");
  if (a->kv_dtype != BLEND_BF16 && a->kv_dtype != BLEND_F32) return fail(BLEND_EINVAL, "kv_dtype");
  if (a->rows_min < 0 || a->min_sep_len < -1 || a->force_class < 0 || a->force_class > 2 ||
      a->split_tokens < 0 || a->num_sms < 0 || a->dense_split < 0 || a->split_waste < 0)
    return fail(BLEND_EINVAL, "rows_min/min_sep_len/force_class/split_tokens/num_sms");
  if (a->n_req < 1) return fail(BLEND_EINVAL, "n_req must be >= 1");
  if (!a->tok_off || !a->tokens || !a->q_len || !a->prompt_len || !a->out_len)
    return fail(BLEND_EINVAL, "NULL input array");
  if (a->tok_off[0] != 0) return fail(BLEND_EMALFORMED, "tok_off[0] must be 0");
  for (int32_t r = 0; r < a->n_req; ++r) {
    int64_t n = a->tok_off[r + 1] - a->tok_off[r];
    if (n < 1) return fail(BLEND_EMALFORMED, "request %d: empty path", r);
    if (n > INT32_MAX / 2) return fail(BLEND_EMALFORMED, "request %d: path too long", r);
    if (a->q_len[r] < 1 || a->q_len[r] > n) return fail(BLEND_EMALFORMED, "request %d: q_len out of range", r);
    if (a->prompt_len[r] < 0 || a->out_len[r] < 0)
      return fail(BLEND_EMALFORMED, "request %d: negative prompt/out length", r);
  }
  int64_t tot = a->tok_off[a->n_req];
  for (int64_t i = 0; i < tot; ++i)
    if (a->tokens[i] < 0) return fail(BLEND_EMALFORMED, "negative token id at %lld", (long long)i);
  return BLEND_OK;
}

int build_descriptors(blend_tree* t);
int build_plan(blend_tree* t);
bool relocation_groups(blend_tree* t, int64_t split_waste);

int build_impl(const blend_build_args* a, blend_tree** out) {
  int st = validate(a);
  if (st) return st;
  blend_tree* t = new (std::nothrow) blend_tree();
  if (!t) return fail(BLEND_ENOMEM, "out of host memory");
  try {
    const int32_t R = a->n_req;
    t->n_req = R;
    t->tok_off.assign(a->tok_off, a->tok_off + R + 1);
    t->tokens.assign(a->tokens, a->tokens + a->tok_off[R]);
    t->q_len.assign(a->q_len, a->q_len + R);
    t->prompt_len.assign(a->prompt_len, a->prompt_len + R);
    t->out_len.assign(a->out_len, a->out_len + R);
    if (a->global_id) t->global_id.assign(a->global_id, a->global_id + R);
    else {
      t->global_id.resize(R);
      for (int32_t r = 0; r < R; ++r) t->global_id[r] = r;
    }
    if (a->free_pages) {
      t->has_free = true;
      t->free_pages.assign(a->free_pages, a->free_pages + std::max<int64_t>(0, a->n_free_pages));
    }
    t->args = *a;
    t->args.tok_off = t->tok_off.data();
    t->args.tokens = t->tokens.data();
    t->args.q_len = t->q_len.data();
    t->args.prompt_len = t->prompt_len.data();
    t->args.out_len = t->out_len.data();
    t->args.global_id = t->global_id.data();
    t->args.free_pages = t->has_free ? t->free_pages.data() : nullptr;
    t->args.n_free_pages = t->has_free ? (int64_t)t->free_pages.size() : 0;
    t->rows_min = a->rows_min == 0 ? 128 : a->rows_min;
    t->min_sep_len = a->min_sep_len < 0 ? 128 : a->min_sep_len;
    t->force_class = a->force_class;
    t->req_group.assign(R, 0);
    st = build_descriptors(t);
    // Alg. 2 (conditional node splitting): relocate outlier subtrees of the sorted tree
    // and rebuild with each relocated subtree in its own root-level group
    if (!st && a->split_waste > 0 && relocation_groups(t, a->split_waste)) st = build_descriptors(t);
    if (!st) st = build_plan(t);
  } catch (const std::bad_alloc&) {
    st = fail(BLEND_ENOMEM, "out of host memory");
  }
  if (st) {
    delete t;
    return st;
  }
  *out = t;
  return BLEND_OK;
}

int build_descriptors(blend_tree* t) {
  const blend_build_args& a = t->args;
  const int32_t R = t->n_req;
  const int32_t* tok = t->tokens.data();
  const int64_t* off = t->tok_off.data();

  // ---- 1. radix trie by insertion (a node boundary at every divergence and every request end)
  std::vector<TNode> nd;
  nd.reserve(2 * R + 16);
  std::vector<std::vector<int32_t>> ends;
  std::unordered_map<uint64_t, int32_t> child;
  child.reserve(4 * R + 16);
  std::vector<int32_t> end_node(R);
  for (int32_t r = 0; r < R; ++r) {
    const int32_t* P = tok + off[r];
    const int32_t n = int32_t(off[r + 1] - off[r]);
    // the root of relocation group g is the pseudo-parent -1 - g: relocated requests
    // never share a node with another group (Alg. 2 duplicates their prefix)
    int32_t node = -1 - t->req_group[r], pos = 0;
    for (;;) {
      auto it = child.find(ckey(node, P[pos]));
      if (it == child.end()) {
        int32_t id = (int32_t)nd.size();
        nd.push_back({pos, n - pos, r, node});
        ends.emplace_back();
        ends.back().push_back(r);
        child.emplace(ckey(node, P[pos]), id);
        end_node[r] = id;
        break;
      }
      int32_t c = it->second;
      const int32_t* seg = tok + off[nd[c].ref] + nd[c].start;
      int32_t L = std::min(nd[c].len, n - pos);
      int32_t k = 0;
      while (k < L && seg[k] == P[pos + k]) ++k;
      if (k < nd[c].len) {  // split c at k
        int32_t u = (int32_t)nd.size();
        nd.push_back({nd[c].start, k, nd[c].ref, node});
        ends.emplace_back();
        it->second = u;
        int32_t next_tok = seg[k];
        nd[c].start += k;
        nd[c].len -= k;
        nd[c].parent = u;
        child.emplace(ckey(u, next_tok), c);
        c = u;
      }
      node = c;
      pos += k;
      if (pos == n) {
        ends[node].push_back(r);
        end_node[r] = node;
        break;
      }
    }
  }
  const int32_t NN = (int32_t)nd.size();
  std::vector<std::vector<int32_t>> kids(NN);
  std::vector<int32_t> tops;
  for (int32_t i = 0; i < NN; ++i) {
    if (nd[i].parent < 0) tops.push_back(i);
    else kids[nd[i].parent].push_back(i);
  }

  // ---- 2. subtree aggregates (post-order) and exact keys
  std::vector<int32_t> post;
  post.reserve(NN);
  {
    std::vector<std::pair<int32_t, int32_t>> st;
    for (int32_t tp : tops) {
      st.push_back({tp, 0});
      while (!st.empty()) {
        auto& f = st.back();
        if (f.second < (int32_t)kids[f.first].size()) {
          int32_t c = kids[f.first][f.second++];
          st.push_back({c, 0});
        } else {
          post.push_back(f.first);
          st.pop_back();
        }
      }
    }
  }
  std::vector<int32_t> nreq(NN, 0), minid(NN, INT32_MAX);
  std::vector<int64_t> maxP(NN, -1);
  std::vector<u128> sum_p2(NN, 0), sum_mu(NN, 0), sum_extra(NN, 0), desc_c(NN, 0);
  auto clampc = [](int64_t v, int64_t hi) -> int64_t { return v < 0 ? 0 : (v > hi ? hi : v); };
  for (int32_t x : post) {
    for (int32_t r : ends[x]) {
      nreq[x] += 1;
      minid[x] = std::min(minid[x], r);
      int64_t p = t->prompt_len[r], d = t->out_len[r], n = off[r + 1] - off[r];
      maxP[x] = std::max(maxP[x], p);
      sum_p2[x] += (u128)p * (u128)p;
      sum_mu[x] += (u128)p * (u128)d + (u128)d * (u128)(d + 1) / 2;
      sum_extra[x] += (u128)(p > n ? p - n : 0) + (u128)d;
    }
    for (int32_t c : kids[x]) {
      nreq[x] += nreq[c];
      minid[x] = std::min(minid[x], minid[c]);
      maxP[x] = std::max(maxP[x], maxP[c]);
      sum_p2[x] += sum_p2[c];
      sum_mu[x] += sum_mu[c];
      sum_extra[x] += sum_extra[c];
      desc_c[x] += desc_c[c] + (u128)clampc(maxP[c] - nd[c].start, nd[c].len);
    }
  }
  std::vector<u128> CU(NN), MU(NN);
  const u128 Pm = (u128)(uint64_t)a.model_params, HL4 = (u128)4 * (u128)(uint32_t)a.hidden * (u128)(uint32_t)a.layers;
  for (int32_t x = 0; x < NN; ++x) {
    u128 G = desc_c[x] + sum_extra[x];
    for (int32_t y = x; y >= 0; y = nd[y].parent) G += (u128)clampc(maxP[x] - nd[y].start, nd[y].len);
    CU[x] = 2 * Pm * G + HL4 * sum_p2[x];
    MU[x] = sum_mu[x];
  }

  // ---- 3. Alg. 1: sort children of every node (and the forest) by rho descending
  auto before = [&](int32_t x, int32_t y) -> bool {
    auto b = [&](int32_t a_, int32_t b_) -> bool {
      if (MU[a_] == 0 && MU[b_] > 0) return true;
      if (MU[a_] == 0 || MU[b_] == 0) return false;
      return gt256(mul_full(CU[a_], MU[b_]), mul_full(CU[b_], MU[a_]));
    };
    if (b(x, y)) return true;
    if (b(y, x)) return false;
    return minid[x] < minid[y];
  };
  std::sort(tops.begin(), tops.end(), before);
  for (auto& v : kids) std::sort(v.begin(), v.end(), before);

  // ---- 4. preorder numbering and request DFS order
  std::vector<int32_t> order;
  order.reserve(NN);
  std::vector<int32_t> dfs;
  dfs.reserve(R);
  {
    std::vector<int32_t> st(tops.rbegin(), tops.rend());
    while (!st.empty()) {
      int32_t x = st.back();
      st.pop_back();
      order.push_back(x);
      for (int32_t r : ends[x]) dfs.push_back(r);   // inserted in ascending r
      for (auto it = kids[x].rbegin(); it != kids[x].rend(); ++it) st.push_back(*it);
    }
  }
  std::vector<int32_t> nid(NN);
  for (int32_t i = 0; i < NN; ++i) nid[order[i]] = i;

  t->n_nodes = NN;
  t->node_parent.resize(NN);
  t->node_start.resize(NN);
  t->node_len.resize(NN);
  t->node_first_req.resize(NN);
  t->node_nreq.resize(NN);
  t->node_class.assign(NN, 0);
  t->node_key_cu.resize(2 * NN);
  t->node_key_mu.resize(2 * NN);
  t->cu.resize(NN);
  t->mu.resize(NN);
  t->node_end_off.assign(NN + 1, 0);
  for (int32_t i = 0; i < NN; ++i) {
    int32_t x = order[i];
    t->node_parent[i] = nd[x].parent < 0 ? -1 : nid[nd[x].parent];
    t->node_start[i] = nd[x].start;
    t->node_len[i] = nd[x].len;
    t->node_first_req[i] = minid[x];
    t->node_nreq[i] = nreq[x];
    t->cu[i] = CU[x];
    t->mu[i] = MU[x];
    t->node_key_cu[2 * i] = (uint64_t)CU[x];
    t->node_key_cu[2 * i + 1] = (uint64_t)(CU[x] >> 64);
    t->node_key_mu[2 * i] = (uint64_t)MU[x];
    t->node_key_mu[2 * i + 1] = (uint64_t)(MU[x] >> 64);
    t->node_end_off[i + 1] = t->node_end_off[i] + (int32_t)ends[x].size();
  }
  t->node_end_req.resize(R);
  for (int32_t i = 0; i < NN; ++i) {
    const auto& e = ends[order[i]];
    std::copy(e.begin(), e.end(), t->node_end_req.begin() + t->node_end_off[i]);
  }
  t->dfs_order = dfs;
  t->req_dfs_rank.resize(R);
  for (int32_t k = 0; k < R; ++k) t->req_dfs_rank[dfs[k]] = k;

  // ---- 5. pages: nodes in id order take ceil(len/ps) consecutive free-list entries
  const int32_t ps = a.page_size;
  t->node_page_off.assign(NN + 1, 0);
  for (int32_t i = 0; i < NN; ++i) t->node_page_off[i + 1] = t->node_page_off[i] + (t->node_len[i] + ps - 1) / ps;
  const int64_t npages = t->node_page_off[NN];
  t->page_table.resize(npages);
  if (t->has_free) {
    if ((int64_t)t->free_pages.size() < npages) return fail(BLEND_ENOSPC, "too few free pages: need %lld", (long long)npages);
    std::vector<int32_t> chk(t->free_pages.begin(), t->free_pages.begin() + npages);
    std::sort(chk.begin(), chk.end());
    if (npages && chk[0] < 0) return fail(BLEND_EINVAL, "negative free page id");
    for (int64_t i = 1; i < npages; ++i)
      if (chk[i] == chk[i - 1]) return fail(BLEND_EINVAL, "duplicate free page id %d", chk[i]);
    std::copy(t->free_pages.begin(), t->free_pages.begin() + npages, t->page_table.begin());
  } else {
    if (npages > INT32_MAX) return fail(BLEND_ENOSPC, "too many pages");
    for (int64_t i = 0; i < npages; ++i) t->page_table[i] = (int32_t)i;
  }
  t->max_page = -1;
  for (int32_t pg : t->page_table) t->max_page = std::max(t->max_page, pg);

  // ---- 6. request paths, classes
  const int32_t g = a.num_q_heads / a.num_kv_heads;
  t->req_path_off.assign(R + 1, 0);
  t->req_path_nodes.clear();
  std::vector<int32_t> chain;
  for (int32_t r = 0; r < R; ++r) {
    chain.clear();
    for (int32_t y = end_node[r]; y >= 0; y = nd[y].parent) chain.push_back(nid[y]);
    t->req_path_off[r + 1] = t->req_path_off[r] + (int64_t)chain.size();
    t->req_path_nodes.insert(t->req_path_nodes.end(), chain.rbegin(), chain.rend());
  }
  t->req_q_off.assign(R + 1, 0);
  t->req_class.assign(R, 0);
  for (int32_t r = 0; r < R; ++r) {
    t->req_q_off[r + 1] = t->req_q_off[r] + t->q_len[r];
    t->req_class[r] = (int64_t)t->q_len[r] * g >= t->rows_min ? 1 : 0;
  }
  std::vector<int64_t> small_q(NN, 0);
  for (int32_t r = 0; r < R; ++r)
    if (!t->req_class[r])
      for (int64_t k = t->req_path_off[r]; k < t->req_path_off[r + 1]; ++k) small_q[t->req_path_nodes[k]] += t->q_len[r];
  for (int32_t i = 0; i < NN; ++i) {
    if (t->force_class == 2 || t->node_nreq[i] < 2) continue;
    if (t->force_class == 1) {
      t->node_class[i] = 1;
      continue;
    }
    if ((int64_t)g * small_q[i] >= t->rows_min && t->node_len[i] >= t->min_sep_len) t->node_class[i] = 1;
  }
  return BLEND_OK;
}

// Alg. 2, conditional node splitting (the algorithm body is missing, P:353,
// DESIGN.md reading #24): a child c of a node with >= 2 children is an outlier when its
// density lies strictly on the other side of the root density rho(rt) than the strict
// majority of its siblings' requests (a sibling subtree's |A| requests count on the side
// of its own density); it is relocated (its prefix duplicated) iff the prefix it shares,
// start(c) tokens, is <= split_waste.  Relocated subtrees are not searched further.
// Sets req_group (k >= 1: the k-th relocated node in preorder); false if none moved.
bool relocation_groups(blend_tree* t, int64_t split_waste) {
  const int32_t NN = t->n_nodes, R = t->n_req;
  u128 cu_rt = 0, mu_rt = 0;
  std::vector<std::vector<int32_t>> kids(NN);
  for (int32_t i = 0; i < NN; ++i) {
    if (t->node_parent[i] < 0) {
      cu_rt += t->cu[i];
      mu_rt += t->mu[i];
    } else {
      kids[t->node_parent[i]].push_back(i);
    }
  }
  auto side = [&](u128 cu, u128 mu) -> int {   // sign(cu / mu - cu_rt / mu_rt), mu = 0 -> +inf
    if (mu == 0) return (cu > 0 || mu_rt > 0) ? 1 : 0;
    const U256 a = mul_full(cu, mu_rt), b = mul_full(cu_rt, mu);
    return gt256(a, b) ? 1 : (gt256(b, a) ? -1 : 0);
  };
  std::vector<char> moved(NN, 0), blocked(NN, 0);
  bool any = false;
  for (int32_t x = 0; x < NN; ++x) {   // preorder: a parent precedes its children
    if (t->node_parent[x] >= 0 && (blocked[t->node_parent[x]] || moved[t->node_parent[x]])) blocked[x] = 1;
    if (blocked[x] || moved[x] || kids[x].size() < 2) continue;
    int64_t up = 0, down = 0;   // requests of the children on each side of rho(rt)
    std::vector<int> sd(kids[x].size());
    for (size_t i = 0; i < kids[x].size(); ++i) {
      const int32_t c = kids[x][i];
      sd[i] = side(t->cu[c], t->mu[c]);
      if (sd[i] > 0) up += t->node_nreq[c];
      if (sd[i] < 0) down += t->node_nreq[c];
    }
    for (size_t i = 0; i < kids[x].size(); ++i) {
      const int32_t c = kids[x][i];
      const int64_t u = up - (sd[i] > 0 ? t->node_nreq[c] : 0), dn = down - (sd[i] < 0 ? t->node_nreq[c] : 0);
      const int sc = sd[i], ss = (u > dn) - (u < dn);
      if (sc != 0 && ss != 0 && sc != ss && (int64_t)t->node_start[c] <= split_waste) {
        moved[c] = 1;
        any = true;
      }
    }
  }
  if (!any) return false;
  std::vector<int32_t> gid(NN, 0);
  int32_t k = 0;
  for (int32_t x = 0; x < NN; ++x)
    if (moved[x]) gid[x] = ++k;
  for (int32_t r = 0; r < R; ++r) {
    t->req_group[r] = 0;
    for (int64_t p = t->req_path_off[r]; p < t->req_path_off[r + 1]; ++p)
      if (gid[t->req_path_nodes[p]]) {
        t->req_group[r] = gid[t->req_path_nodes[p]];
        break;
      }
  }
  return true;
}

// ---------------------------------------------------------------------------
// Work plan
// ---------------------------------------------------------------------------
struct Item {
  std::vector<int32_t> toks;           // global token rows, item-row order
  std::vector<blend::KvEntry> ents;    // ascending positions
  bool dense = false;
};

void node_entries(const blend_tree* t, int32_t node, std::vector<blend::KvEntry>& out) {
  const int32_t ps = t->args.page_size;
  const int32_t start = t->node_start[node], len = t->node_len[node];
  for (int64_t i = t->node_page_off[node]; i < t->node_page_off[node + 1]; ++i) {
    int32_t k = int32_t(i - t->node_page_off[node]);
    int32_t cnt = std::min(ps, len - k * ps);
    int32_t page = t->page_table[i];
    if (ps <= blend::ENTRY_MAX) {
      out.push_back({page, 0, start + k * ps, cnt});
    } else {
      for (int32_t h = 0; h * blend::ENTRY_MAX < cnt; ++h)
        out.push_back({page, h * blend::ENTRY_MAX, start + k * ps + h * blend::ENTRY_MAX,
                       std::min(blend::ENTRY_MAX, cnt - h * blend::ENTRY_MAX)});
    }
  }
}

int build_plan(blend_tree* t) {
  const blend_build_args& a = t->args;
  const int32_t R = t->n_req, NN = t->n_nodes, Hkv = a.num_kv_heads;
  const int32_t g = a.num_q_heads / a.num_kv_heads;
  const int32_t num_sms = a.num_sms ? a.num_sms : 148;
  const int64_t T = t->req_q_off[R];
  if (T > INT32_MAX / 2) return fail(BLEND_EINVAL, "too many query tokens");

  std::vector<int32_t> tok_pos(T);
  for (int32_t r = 0; r < R; ++r) {
    int32_t n = int32_t(t->tok_off[r + 1] - t->tok_off[r]);
    for (int32_t q = 0; q < t->q_len[r]; ++q) tok_pos[t->req_q_off[r] + q] = n - t->q_len[r] + q;
  }
  auto sep_for = [&](int32_t node, int32_t r) {
    return t->node_class[node] && (!t->req_class[r] || t->force_class == 1);
  };

  // ---- items: one per SEPARATE node (its users' rows), one per request (remaining nodes)
  std::vector<Item> items;
  std::vector<int32_t> sep_item(NN, -1);
  for (int32_t i = 0; i < NN; ++i)
    if (t->node_class[i]) {
      sep_item[i] = (int32_t)items.size();
      items.emplace_back();
      node_entries(t, i, items.back().ents);
    }
  for (int32_t k = 0; k < R; ++k) {
    int32_t r = t->dfs_order[k];
    for (int64_t p = t->req_path_off[r]; p < t->req_path_off[r + 1]; ++p) {
      int32_t node = t->req_path_nodes[p];
      if (sep_for(node, r)) {
        auto& it = items[sep_item[node]];
        for (int32_t q = 0; q < t->q_len[r]; ++q) it.toks.push_back(int32_t(t->req_q_off[r] + q));
      }
    }
  }
  // A SEPARATE item's rows may come in any order (every row carries its own position
  // and partmap slot): ascending q rows make the users' tokens consecutive wherever the
  // caller keeps them together, so the dense kernel loads such Q tiles with whole TMA
  // boxes instead of one box per token.
  for (auto& it : items) std::sort(it.toks.begin(), it.toks.end());
  for (int32_t k = 0; k < R; ++k) {
    int32_t r = t->dfs_order[k];
    Item it;
    for (int64_t p = t->req_path_off[r]; p < t->req_path_off[r + 1]; ++p) {
      int32_t node = t->req_path_nodes[p];
      if (!sep_for(node, r)) node_entries(t, node, it.ents);
    }
    if (it.ents.empty()) continue;
    for (int32_t q = 0; q < t->q_len[r]; ++q) it.toks.push_back(int32_t(t->req_q_off[r] + q));
    items.push_back(std::move(it));
  }
  // drop SEPARATE items nobody uses (cannot happen by the class rule, kept for safety)
  items.erase(std::remove_if(items.begin(), items.end(), [](const Item& x) { return x.toks.empty(); }), items.end());
  for (auto& it : items) it.dense = (int64_t)it.toks.size() * g >= t->rows_min;

  const int32_t tile_d = g <= blend::DENSE_ROWS ? (blend::DENSE_ROWS / g) * g : blend::DENSE_ROWS;
  const int32_t tile_s = g <= blend::STREAM_ROWS ? (blend::STREAM_ROWS / g) * g : blend::STREAM_ROWS;
  auto ntiles = [&](const Item& it) {
    int64_t rows = (int64_t)it.toks.size() * g;
    int32_t tr = it.dense ? tile_d : tile_s;
    return (rows + tr - 1) / tr;
  };

  // ---- split-KV decisions (plan only; not part of the bit-exact contract)
  int64_t base_d = 0, base_s = 0, work_s = 0;
  double flops_d = 0.0, bytes_s = 0.0;
  const int kvb = a.kv_dtype == BLEND_BF16 ? 2 : 4;
  for (auto& it : items) {
    int64_t u = ntiles(it) * Hkv;
    int64_t kv = 0;
    for (auto& e : it.ents) kv += e.count;
    if (it.dense) {
      base_d += u;
      flops_d += 4.0 * a.head_dim * (double)it.toks.size() * a.num_q_heads * (double)kv;
    } else {
      base_s += u;
      work_s += u * kv;
      bytes_s += (double)u * kv * a.head_dim * 2 * kvb;
    }
  }
  int64_t chunk_s = INT64_MAX;
  if (a.split_tokens > 0) chunk_s = a.split_tokens;
  else if (base_s > 0 && base_s < 8LL * num_sms) {
    chunk_s = std::max<int64_t>(512, (work_s + 8LL * num_sms - 1) / (8LL * num_sms));
    chunk_s = (chunk_s + 63) / 64 * 64;
  }
  // dense split-KV: the dense grid overlaps the streaming grid (PDL), so give it the
  // share of the SMs proportional to its estimated time (NEXT-1, the paper's resource
  // overlap f = max, §2.4) and split its items until that share is filled.
  // Rates are planning constants measured on B200 for the two kernels (~800 TFLOP/s
  // dense, ~6 TB/s streaming; a 250 TFLOP/s estimate gave the dense pass twice the SMs
  // the streaming pass could spare: C2 47.3 us with 64 dense CTAs, 43.7 us with 32).
  // When the dense pass alone would fill the GPU and both passes are substantial, cap
  // its grid so the overlapped streaming grid starts on the remaining SMs at once.  The
  // cap is the dense pass's share of the SM-time: a = (dense time on the whole GPU) x
  // SMs, b = streaming bytes / (per-SM streaming rate), D = SMs x a / (a + b), so that
  // both grids finish together.  On fewer SMs the streaming pass is bound by its
  // consumer warps (~BLEND_STREAM_SM_GBS per SM, well under an SM's share of HBM), not
  // by HBM.  Rates: ~690 TFLOP/s dense (round-1), 68 GB/s per SM streaming (one
  // consumer warp per SM streams C4 at 17 GB/s, round 2).
  t->dense_ctas = 0;
  double cap_a = 0.0, cap_b = 0.0;   // SM-time of the dense and the streaming pass (see the key-split units below)
  if (base_d >= num_sms && flops_d > 0.0 && bytes_s > 0.0) {
    const double td = flops_d / 690e12, ts = bytes_s / 6.9e12;
    if (td > 0.2 * (td + ts) && ts > 0.2 * (td + ts)) {
      const double a = td * num_sms, b = bytes_s / (BLEND_STREAM_SM_GBS * 1e9);
      t->dense_ctas = (int32_t)(num_sms * a / (a + b) + 0.5);
      cap_a = a;
      cap_b = b;
    }
  }
  int64_t dsplit = 1;
  if (a.dense_split > 0) dsplit = a.dense_split;
  else if (base_d > 0 && base_d < num_sms) {
    const double t_d = flops_d / 800e12, t_s = bytes_s / 6e12;
    const double share = t_d / (t_d + t_s);
    const int64_t dense_sms = std::max<int64_t>(1, (int64_t)(share * num_sms + 0.5));
    dsplit = std::max<int64_t>(1, (dense_sms + base_d / 2) / base_d);
    // When the dense pass is comparable to the streaming pass (a data-parallel shard of
    // a long-document batch: C5 split over 4-8 GPUs), its few long units would run on a
    // fraction of the SMs long after the streaming grid has finished (the SM split of the
    // overlap cannot be rebalanced at run time): split them to fill the GPU instead
    // (measured, C5 rank of 8: dense 0.45 -> 0.13 ms, step 0.49 -> 0.34 ms with 4 splits).
    // (Only when the units would occupy at most half of the SMs; the split is the smallest
    // that minimises the wave-quantised dense time ceil(base_d s / num_sms) / s.)
    if (t_d >= 0.5 * t_s && 2 * base_d <= num_sms) {
      double best = 1.0;
      for (int64_t s_ = 2; s_ <= 8; ++s_) {
        const double tq = (double)((base_d * s_ + num_sms - 1) / num_sms) / (double)s_;
        if (tq < best - 1e-9) {
          best = tq;
          dsplit = std::max<int64_t>(dsplit, s_);
        }
      }
    }
  } else if (base_d > 0) {
    // more units than SMs: split long items so the last wave of persistent CTAs is full
    // (e.g. 256 units of a 31K-token document on 148 SMs -> 4 splits, 99% wave fill)
    int64_t n_dense_items = 0, kv_dense = 0;
    for (auto& it : items)
      if (it.dense) {
        ++n_dense_items;
        for (auto& e : it.ents) kv_dense += e.count;
      }
    const int64_t avg_kv = kv_dense / std::max<int64_t>(1, n_dense_items);
    auto fill = [&](int64_t s_) {   // wave fill with the per-item cap min(s, kv / 256) used below
      int64_t units = 0;
      for (auto& it : items)
        if (it.dense) {
          int64_t kv = 0;
          for (auto& e : it.ents) kv += e.count;
          units += ntiles(it) * Hkv * std::max<int64_t>(1, std::min<int64_t>(s_, kv / 256));
        }
      const int64_t waves = (units + num_sms - 1) / num_sms;
      return (double)units / (double)(waves * num_sms);
    };
    double best = fill(1);
    for (int64_t s_ = 2; s_ <= 8 && avg_kv / s_ >= 2048; ++s_)
      if (fill(s_) > best + 0.02) {
        best = fill(s_);
        dsplit = s_;
      }
  }

  // Streaming tail balance: units go out longest first to R = 4 x num_sms rings; when
  // the last round would be less than half full, the shortest streaming items are split
  // in two (by keys), so that round consists of half-length units and finishes in about
  // half the time (C2: 2048 units on 592 rings).  Plan only, outside the bit-exact
  // contract; the extra partials are merged like any split-KV source.
  std::vector<char> split_tail(items.size(), 0);
  if (chunk_s == INT64_MAX && a.split_tokens == 0) {
    const int64_t R = 4LL * num_sms, rem = base_s % R;
    if (base_s >= R && rem > 0 && rem <= R / 2) {
      std::vector<size_t> order;
      for (size_t ii = 0; ii < items.size(); ++ii)
        if (!items[ii].dense && items[ii].ents.size() >= 2) order.push_back(ii);
      std::stable_sort(order.begin(), order.end(),
                       [&](size_t x, size_t y) { return items[x].ents.size() < items[y].ents.size(); });
      int64_t covered = 0;
      for (size_t ii : order) {
        if (covered >= rem) break;
        split_tail[ii] = 1;
        covered += ntiles(items[ii]) * Hkv;
      }
    }
  }

  std::vector<std::vector<int32_t>> split_b(items.size());   // entry boundaries per item
  for (size_t ii = 0; ii < items.size(); ++ii) {
    auto& it = items[ii];
    auto& b = split_b[ii];
    b.push_back(0);
    const int32_t E = (int32_t)it.ents.size();
    if (it.dense) {
      int64_t kv = 0;
      for (auto& e : it.ents) kv += e.count;
      int64_t ns = std::max<int64_t>(1, std::min<int64_t>(dsplit, kv / 256));
      int64_t acc = 0, next = 1;
      for (int32_t e = 0; e < E && next < ns; ++e) {
        acc += it.ents[e].count;
        if (acc * ns >= next * kv && e + 1 < E) {
          b.push_back(e + 1);
          ++next;
        }
      }
    } else if (chunk_s != INT64_MAX) {
      int64_t acc = 0;
      for (int32_t e = 0; e < E; ++e) {
        acc += it.ents[e].count;
        if (acc >= chunk_s && e + 1 < E) {
          b.push_back(e + 1);
          acc = 0;
        }
      }
    } else if (split_tail[ii]) {
      int64_t kv = 0, acc = 0;
      for (auto& e : it.ents) kv += e.count;
      for (int32_t e = 0; e + 1 < E; ++e) {
        acc += it.ents[e].count;
        if (2 * acc >= kv) {
          b.push_back(e + 1);
          break;
        }
      }
    }
    b.push_back(E);
  }

  // ---- sources per token: (key start, partmap index); partmap per (item, split)
  std::vector<int32_t> item_tok_off(items.size() + 1, 0);
  for (size_t ii = 0; ii < items.size(); ++ii) item_tok_off[ii + 1] = item_tok_off[ii] + (int32_t)items[ii].toks.size();
  std::vector<std::vector<int32_t>> pm_base(items.size());
  int64_t pm_size = 0;
  for (size_t ii = 0; ii < items.size(); ++ii)
    for (size_t s = 0; s + 1 < split_b[ii].size(); ++s) {
      pm_base[ii].push_back((int32_t)pm_size);
      pm_size += (int64_t)items[ii].toks.size();
    }
  if (pm_size > INT32_MAX / 2) return fail(BLEND_EINVAL, "plan too large");
  std::vector<int32_t> partmap(pm_size, blend::PM_SKIP);
  std::vector<int32_t> nsrc(T, 0);
  struct Src {
    int32_t tok, key_start, pm;
  };
  std::vector<Src> srcs;
  for (size_t ii = 0; ii < items.size(); ++ii) {
    auto& it = items[ii];
    for (size_t s = 0; s + 1 < split_b[ii].size(); ++s) {
      int32_t ks = it.ents[split_b[ii][s]].pos0;
      for (size_t i = 0; i < it.toks.size(); ++i) {
        int32_t tk = it.toks[i];
        if (ks <= tok_pos[tk]) {
          nsrc[tk] += 1;
          srcs.push_back({tk, ks, pm_base[ii][s] + (int32_t)i});
        }
      }
    }
  }
  for (int64_t tk = 0; tk < T; ++tk)
    if (nsrc[tk] < 1) return fail(BLEND_EMALFORMED, "internal: token %lld has no source", (long long)tk);
  std::stable_sort(srcs.begin(), srcs.end(), [](const Src& x, const Src& y) {
    return x.tok != y.tok ? x.tok < y.tok : x.key_start < y.key_start;
  });
  // Merge lists, ascending key start (reading #17): list m holds the partial rows
  // merge_off[m] .. merge_off[m+1]-1 in that order, so the merge kernel reads partial
  // row s for list entry s without an index lookup.
  std::vector<int32_t> merge_tok, merge_off{0};
  int64_t prow = 0;
  for (size_t i = 0; i < srcs.size();) {
    size_t j = i;
    while (j < srcs.size() && srcs[j].tok == srcs[i].tok) ++j;
    if (j - i == 1) {
      partmap[srcs[i].pm] = blend::PM_DIRECT;
    } else {
      merge_tok.push_back(srcs[i].tok);
      for (size_t k = i; k < j; ++k) partmap[srcs[k].pm] = (int32_t)prow++;
      merge_off.push_back((int32_t)prow);
    }
    i = j;
  }
  const int32_t n_merge = (int32_t)merge_tok.size();
  t->merge_nsrc = 0;
  if (n_merge > 0) {
    const int32_t n0 = merge_off[1] - merge_off[0];
    bool uni = true;
    for (int32_t m = 1; m < n_merge && uni; ++m) uni = merge_off[m + 1] - merge_off[m] == n0;
    if (uni) t->merge_nsrc = n0;
  }
  if (prow > INT32_MAX / 2) return fail(BLEND_EINVAL, "too many partial rows");

  // ---- entries and units
  std::vector<blend::KvEntry> ents;
  std::vector<int32_t> item_ent_off(items.size() + 1, 0);
  for (size_t ii = 0; ii < items.size(); ++ii) {
    item_ent_off[ii] = (int32_t)ents.size();
    ents.insert(ents.end(), items[ii].ents.begin(), items[ii].ents.end());
  }
  item_ent_off[items.size()] = (int32_t)ents.size();
  std::vector<blend::Unit> dunits, sunits;
  int64_t dense_kv = 0, stream_kv = 0;
  for (size_t ii = 0; ii < items.size(); ++ii) {
    auto& it = items[ii];
    const int64_t rows = (int64_t)it.toks.size() * g;
    const int32_t tr = it.dense ? tile_d : tile_s;
    for (int64_t rb = 0; rb < rows; rb += tr) {
      int32_t nr = (int32_t)std::min<int64_t>(tr, rows - rb);
      int32_t maxpos = INT32_MIN;   // SEPARATE items mix requests: positions are not sorted
      for (int64_t tl = rb / g; tl <= (rb + nr - 1) / g; ++tl) maxpos = std::max(maxpos, tok_pos[it.toks[tl]]);
      int32_t trunc = 0;   // entries with pos0 <= maxpos (ascending positions)
      while (trunc < (int32_t)it.ents.size() && it.ents[trunc].pos0 <= maxpos) ++trunc;
      for (size_t s = 0; s + 1 < split_b[ii].size(); ++s) {
        int32_t e0 = split_b[ii][s], e1 = std::min(split_b[ii][s + 1], trunc);
        if (e1 <= e0) continue;
        int64_t kv = 0;
        for (int32_t e = e0; e < e1; ++e) kv += it.ents[e].count;
        for (int32_t h = 0; h < Hkv; ++h) {
          blend::Unit u{(int32_t)ii, h, (int32_t)rb, nr, item_ent_off[ii] + e0, item_ent_off[ii] + e1,
                        pm_base[ii][s], item_tok_off[ii]};
          (it.dense ? dunits : sunits).push_back(u);
          (it.dense ? dense_kv : stream_kv) += kv;
        }
      }
    }
  }
  auto by_work = [](const blend::Unit& x, const blend::Unit& y) {
    return (x.entry_end - x.entry_begin) > (y.entry_end - y.entry_begin);
  };
  std::stable_sort(dunits.begin(), dunits.end(), by_work);
  std::stable_sort(sunits.begin(), sunits.end(), by_work);
  t->stream_entries = 0;
  for (const auto& u : sunits) t->stream_entries += u.entry_end - u.entry_begin;

  std::vector<int32_t> item_tokens(item_tok_off.back());
  for (size_t ii = 0; ii < items.size(); ++ii)
    std::copy(items[ii].toks.begin(), items[ii].toks.end(), item_tokens.begin() + item_tok_off[ii]);

  // Dense units whose query tokens are consecutive rows of q (a request's prefill chunk)
  // and whose 128-row tiles hold whole tokens load Q with 3-D TMA boxes {64, g, 128/g}.
  std::vector<int32_t> dqtok(dunits.size(), -1);
  if (blend::DENSE_ROWS % g == 0 && 128 % g == 0)
    for (size_t ui = 0; ui < dunits.size(); ++ui) {
      const blend::Unit& u = dunits[ui];
      const int32_t tl0 = u.row_begin / g, tl1 = (u.row_begin + u.n_rows - 1) / g;
      if (u.row_begin % g) continue;
      const int32_t t0 = item_tokens[u.tok_base + tl0];
      bool consec = true;
      for (int32_t tl = tl0 + 1; tl <= tl1 && consec; ++tl) consec = item_tokens[u.tok_base + tl] == t0 + (tl - tl0);
      if (consec) dqtok[ui] = t0;
    }

  // Key-split units: <= 128 rows (one Q tile) and >= 2 64-key blocks run in dense_ks.cu,
  // where the CTA's two tiles take alternate blocks of the one tile and merge at the end
  // (a separate launch; both lists keep the longest-first order).
  std::vector<blend::Unit> dunits_ks;
  std::vector<int32_t> dqtok_ks;
  {
    const int32_t epb = 64 / std::min<int32_t>(a.page_size, 64);
    std::vector<blend::Unit> keep;
    std::vector<int32_t> keep_q;
    for (size_t ui = 0; ui < dunits.size(); ++ui) {
      const blend::Unit& u = dunits[ui];
      const int32_t nb = (u.entry_end - u.entry_begin + epb - 1) / epb;
      if (u.n_rows <= 128 && nb >= 2 && a.kv_dtype == BLEND_BF16) {
        dunits_ks.push_back(u);
        dqtok_ks.push_back(dqtok[ui]);
      } else {
        keep.push_back(u);
        keep_q.push_back(dqtok[ui]);
      }
    }
    dunits.swap(keep);
    dqtok.swap(keep_q);
  }
  // The key-split units run after the streaming grid (on every SM), so only the two-tile
  // units' share of the dense SM-time is balanced against the streaming pass: a splits by
  // the two lists' block counts weighted with their measured per-block cost (a key-split
  // block, one 128-row tile: 0.54 of a two-tile block pair; C4).
  if (t->dense_ctas > 0 && !dunits_ks.empty() && cap_a > 0.0) {
    const int32_t epb = 64 / std::min<int32_t>(a.page_size, 64);
    double w_d = 0.0, w_k = 0.0;
    for (const auto& u : dunits) w_d += (double)((u.entry_end - u.entry_begin + epb - 1) / epb);
    for (const auto& u : dunits_ks) w_k += 0.54 * (double)((u.entry_end - u.entry_begin + epb - 1) / epb);
    const double a_d = cap_a * w_d / (w_d + w_k);
    t->dense_ctas = std::max<int32_t>(1, (int32_t)(num_sms * a_d / (a_d + cap_b) + 0.5));
  }

  // Per-row descriptors of the streaming units (STREAM_ROWS slots per unit): the
  // kernel gets each row's q/out row, position and partmap target in one load
  // instead of the item_tokens -> tok_pos / partmap chain.
  std::vector<blend::RowDesc> srows(sunits.size() * blend::STREAM_ROWS,
                                    blend::RowDesc{-1, INT32_MIN, blend::PM_SKIP, -1});
  for (size_t ui = 0; ui < sunits.size(); ++ui) {
    const blend::Unit& u = sunits[ui];
    for (int r = 0; r < u.n_rows; ++r) {
      const int32_t ir = u.row_begin + r, tl = ir / g, j = ir % g;
      const int32_t tok = item_tokens[u.tok_base + tl];
      blend::RowDesc& d = srows[ui * blend::STREAM_ROWS + r];
      d.qrow = tok * a.num_q_heads + u.kvh * g + j;
      d.pos = tok_pos[tok];
      d.target = partmap[u.pm_base + tl];
      d.head = u.kvh * g + j;
    }
  }

  // ---- serialise sections (16-byte aligned)
  using namespace blend;
  std::vector<uint8_t>& blob = t->plan_blob;
  blob.clear();
  auto put = [&](int sec, const void* p, size_t elem, size_t n) {
    size_t o = (blob.size() + 15) & ~size_t(15);
    blob.resize(o + elem * n);
    if (n) memcpy(blob.data() + o, p, elem * n);
    t->sec_off[sec] = (int64_t)o;
    t->sec_count[sec] = (int64_t)n;
  };
  put(SEC_TOK_POS, tok_pos.data(), 4, tok_pos.size());
  put(SEC_ITEM_TOK_OFF, item_tok_off.data(), 4, item_tok_off.size());
  put(SEC_ITEM_TOKENS, item_tokens.data(), 4, item_tokens.size());
  put(SEC_ENTRIES, ents.data(), sizeof(KvEntry), ents.size());
  put(SEC_DENSE_UNITS, dunits.data(), sizeof(Unit), dunits.size());
  put(SEC_STREAM_UNITS, sunits.data(), sizeof(Unit), sunits.size());
  put(SEC_PARTMAP, partmap.data(), 4, partmap.size());
  put(SEC_MERGE_TOK, merge_tok.data(), 4, merge_tok.size());
  put(SEC_MERGE_OFF, merge_off.data(), 4, merge_off.size());
  put(SEC_STREAM_ROWS, srows.data(), sizeof(RowDesc), srows.size());
  put(SEC_DENSE_QTOK, dqtok.data(), 4, dqtok.size());
  put(SEC_DENSE_KS, dunits_ks.data(), sizeof(Unit), dunits_ks.size());
  put(SEC_DENSE_KS_QTOK, dqtok_ks.data(), 4, dqtok_ks.size());
  blob.resize((blob.size() + 255) & ~size_t(255));

  t->n_partial_rows = prow;
  const size_t hq = a.num_q_heads, D = a.head_dim;
  size_t o_bytes = ((size_t)prow * hq * D * 4 + 255) & ~size_t(255);
  // partials o | lse | unit counter of the streaming pass (256 B)
  t->workspace_bytes = o_bytes + (((size_t)prow * hq * 4 + 255) & ~size_t(255)) + 256;
  t->info.n_tokens = T;
  t->info.n_items = (int64_t)items.size();
  t->info.n_dense_units = (int64_t)(dunits.size() + dunits_ks.size());
  t->info.n_stream_units = (int64_t)sunits.size();
  t->info.n_partial_rows = prow;
  t->info.n_merge_tokens = (int64_t)merge_tok.size();
  t->info.n_entries = (int64_t)ents.size();
  t->info.dense_kv_tokens = dense_kv;
  t->info.stream_kv_tokens = stream_kv;
  return BLEND_OK;
}

// ---------------------------------------------------------------------------
// Sharder (§7.1)
// ---------------------------------------------------------------------------
int32_t lcp_tokens(const blend_tree* t, int32_t a, int32_t b) {
  const int32_t* A = t->tokens.data() + t->tok_off[a];
  const int32_t* B = t->tokens.data() + t->tok_off[b];
  int32_t n = (int32_t)std::min(t->tok_off[a + 1] - t->tok_off[a], t->tok_off[b + 1] - t->tok_off[b]);
  int32_t k = 0;
  while (k < n && A[k] == B[k]) ++k;
  return k;
}

int shard_impl(const blend_tree* t, int32_t G, int64_t kappa, const int32_t* const* sfree,
               const int64_t* nsfree, int32_t* req_shard, blend_tree** shards) {
  if (!t || !req_shard) return fail(BLEND_EINVAL, "NULL argument");
  if (G < 1) return fail(BLEND_EINVAL, "n_shards must be >= 1");
  if (kappa <= 0) kappa = 213;
  const blend_build_args& a = t->args;
  const int32_t R = t->n_req;
  const i128 D = a.head_dim, Hq = a.num_q_heads, Hkv = a.num_kv_heads, b = a.kv_dtype == BLEND_BF16 ? 2 : 4;
  std::vector<char> touched(t->n_nodes, 0);
  std::vector<i128> S(R + 1, 0);
  for (int32_t k = 0; k < R; ++k) {
    int32_t r = t->dfs_order[k];
    i128 n = t->tok_off[r + 1] - t->tok_off[r], q = t->q_len[r];
    i128 flops = 4 * D * Hq * (q * (n - q) + q * (q + 1) / 2);
    i128 ft = 0;
    for (int64_t p = t->req_path_off[r]; p < t->req_path_off[r + 1]; ++p) {
      int32_t node = t->req_path_nodes[p];
      if (!touched[node]) {
        touched[node] = 1;
        ft += (i128)t->node_len[node] * Hkv * D * 2 * b;
      }
    }
    S[k + 1] = S[k] + flops + (i128)kappa * ft;
  }
  const i128 W = S[R];
  std::vector<int32_t> lcp(R + 1, 0);
  for (int32_t k = 1; k < R; ++k) lcp[k] = lcp_tokens(t, t->dfs_order[k - 1], t->dfs_order[k]);
  std::vector<int32_t> cuts{0};
  for (int32_t i = 1; i < 2 * G; ++i) {
    i128 num = (i128)i * W, den = 2 * (i128)G;
    i128 tau = (num + den - 1) / den;
    int32_t best = -1;
    for (int32_t k = 0; k <= R; ++k) {
      i128 dk = S[k] > tau ? S[k] - tau : tau - S[k];
      if (dk * 32 * G > W) continue;
      if (best < 0) {
        best = k;
        continue;
      }
      i128 db = S[best] > tau ? S[best] - tau : tau - S[best];
      if (lcp[k] < lcp[best] || (lcp[k] == lcp[best] && dk < db)) best = k;
    }
    if (best < 0) {
      i128 bd = -1;
      for (int32_t k = 0; k <= R; ++k) {
        i128 dk = S[k] > tau ? S[k] - tau : tau - S[k];
        if (bd < 0 || dk < bd) {
          bd = dk;
          best = k;
        }
      }
    }
    cuts.push_back(std::max(best, cuts.back()));
  }
  cuts.push_back(R);
  for (int32_t j = 0; j < 2 * G; ++j) {
    int32_t gsh = j < G ? j : 2 * G - 1 - j;
    for (int32_t k = cuts[j]; k < cuts[j + 1]; ++k) req_shard[t->dfs_order[k]] = gsh;
  }
  if (!shards) return BLEND_OK;
  for (int32_t gsh = 0; gsh < G; ++gsh) shards[gsh] = nullptr;
  for (int32_t gsh = 0; gsh < G; ++gsh) {
    std::vector<int32_t> rs;
    for (int32_t r = 0; r < R; ++r)
      if (req_shard[r] == gsh) rs.push_back(r);
    if (rs.empty()) continue;
    std::vector<int64_t> off{0}, gid;
    std::vector<int32_t> toks, q, p, d;
    for (int32_t r : rs) {
      toks.insert(toks.end(), t->tokens.begin() + t->tok_off[r], t->tokens.begin() + t->tok_off[r + 1]);
      off.push_back((int64_t)toks.size());
      q.push_back(t->q_len[r]);
      p.push_back(t->prompt_len[r]);
      d.push_back(t->out_len[r]);
      gid.push_back(t->global_id[r]);
    }
    blend_build_args sa = a;
    sa.n_req = (int32_t)rs.size();
    sa.tok_off = off.data();
    sa.tokens = toks.data();
    sa.q_len = q.data();
    sa.prompt_len = p.data();
    sa.out_len = d.data();
    sa.global_id = gid.data();
    sa.free_pages = sfree ? sfree[gsh] : nullptr;
    sa.n_free_pages = (sfree && nsfree) ? nsfree[gsh] : 0;
    sa.rows_min = t->rows_min;
    sa.min_sep_len = t->min_sep_len;
    int st = build_impl(&sa, &shards[gsh]);
    if (st) {
      for (int32_t k = 0; k < G; ++k) {
        delete shards[k];
        shards[k] = nullptr;
      }
      return st;
    }
  }
  return BLEND_OK;
}

}  // namespace

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" {

const char* blend_last_error(void) { return g_err.c_str(); }
int blend_abi_version(void) { return BLEND_ABI_VERSION; }

int blend_tree_build(const blend_build_args* args, blend_tree** out) {
  if (!out) return fail(BLEND_EINVAL, "out is NULL");
  *out = nullptr;
  return build_impl(args, out);
}

void blend_tree_free(blend_tree* t) { delete t; }

int blend_tree_get_view(const blend_tree* t, blend_tree_view* v) {
  if (!t || !v) return fail(BLEND_EINVAL, "NULL argument");
  v->n_req = t->n_req;
  v->n_nodes = t->n_nodes;
  v->n_pages = t->node_page_off.empty() ? 0 : t->node_page_off.back();
  v->node_parent = t->node_parent.data();
  v->node_start = t->node_start.data();
  v->node_len = t->node_len.data();
  v->node_page_off = t->node_page_off.data();
  v->node_class = t->node_class.data();
  v->node_key_cu = t->node_key_cu.data();
  v->node_key_mu = t->node_key_mu.data();
  v->node_first_req = t->node_first_req.data();
  v->node_nreq = t->node_nreq.data();
  v->page_table = t->page_table.data();
  v->req_path_off = t->req_path_off.data();
  v->req_path_nodes = t->req_path_nodes.data();
  v->req_q_off = t->req_q_off.data();
  v->req_class = t->req_class.data();
  v->req_dfs_rank = t->req_dfs_rank.data();
  v->req_global_id = t->global_id.data();
  v->req_group = t->req_group.data();
  return BLEND_OK;
}

int blend_tree_dump(const blend_tree* t, char* buf, size_t cap, size_t* need) {
  if (!t) return fail(BLEND_EINVAL, "tree is NULL");
  std::string s;
  std::vector<int32_t> depth(t->n_nodes, 0);
  char line[256];
  for (int32_t i = 0; i < t->n_nodes; ++i) {
    int32_t par = t->node_parent[i];
    depth[i] = par < 0 ? 0 : depth[par] + 1;
    s.append(2 * depth[i], ' ');
    snprintf(line, sizeof line, "#%d start=%d len=%d tok=[", i, t->node_start[i], t->node_len[i]);
    s += line;
    const int32_t* P = t->tokens.data() + t->tok_off[t->node_first_req[i]] + t->node_start[i];
    for (int32_t k = 0; k < std::min(8, t->node_len[i]); ++k) {
      if (k) s += ',';
      s += std::to_string(P[k]);
    }
    s += "] cu=" + u128_str(t->cu[i]) + " mu=" + u128_str(t->mu[i]);
    s += t->node_class[i] ? " cls=S" : " cls=F";
    s += " nreq=" + std::to_string(t->node_nreq[i]) + " ends=[";
    for (int32_t k = t->node_end_off[i]; k < t->node_end_off[i + 1]; ++k) {
      if (k > t->node_end_off[i]) s += ',';
      s += std::to_string(t->node_end_req[k]);
    }
    s += "]\n";
  }
  if (need) *need = s.size() + 1;
  if (cap > 0 && buf) {
    size_t n = std::min(cap - 1, s.size());
    memcpy(buf, s.data(), n);
    buf[n] = 0;
  }
  if (cap < s.size() + 1) return fail(BLEND_ENOSPC, "dump buffer too small");
  return BLEND_OK;
}

int blend_shard(const blend_tree* t, int32_t n_shards, int64_t kappa, const int32_t* const* shard_free_pages,
                const int64_t* n_shard_free, int32_t* req_shard, blend_tree** shards) {
  try {
    return shard_impl(t, n_shards, kappa, shard_free_pages, n_shard_free, req_shard, shards);
  } catch (const std::bad_alloc&) {
    return fail(BLEND_ENOMEM, "out of host memory");
  }
}

int blend_plan_get_info(const blend_tree* t, blend_plan_info* info) {
  if (!t || !info) return fail(BLEND_EINVAL, "NULL argument");
  *info = t->info;
  return BLEND_OK;
}

size_t blend_plan_bytes(const blend_tree* t) { return t ? t->plan_blob.size() : 0; }
size_t blend_workspace_bytes(const blend_tree* t) { return t ? t->workspace_bytes : 0; }

// used by the device-side upload (attention.cu)
int blend_internal_plan_image(const blend_tree* t, const void** data, size_t* bytes, const int64_t** off,
                              const int64_t** count) {
  if (!t) return fail(BLEND_EINVAL, "tree is NULL");
  *data = t->plan_blob.data();
  *bytes = t->plan_blob.size();
  *off = t->sec_off;
  *count = t->sec_count;
  return BLEND_OK;
}

int blend_internal_fail(int status, const char* msg) { return fail(status, "%s", msg); }

int64_t blend_internal_partial_rows(const blend_tree* t) { return t ? t->n_partial_rows : 0; }
int64_t blend_internal_stream_entries(const blend_tree* t) { return t ? t->stream_entries : 0; }
int32_t blend_internal_max_page(const blend_tree* t) { return t ? t->max_page : -1; }
int32_t blend_internal_dense_ctas(const blend_tree* t) { return t ? t->dense_ctas : 0; }
int32_t blend_internal_merge_nsrc(const blend_tree* t) { return t ? t->merge_nsrc : 0; }

int blend_internal_tree_dims(const blend_tree* t, int32_t* dims) {
  if (!t) return fail(BLEND_EINVAL, "tree is NULL");
  dims[0] = t->args.num_q_heads;
  dims[1] = t->args.num_kv_heads;
  dims[2] = t->args.head_dim;
  dims[3] = t->args.kv_dtype;
  dims[4] = t->args.page_size;
  return BLEND_OK;
}

}  // extern "C"
