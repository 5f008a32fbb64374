// sched.cpp — the dual-scanner batch former (NEXT-2): turns the density-sorted
// tree of a whole offline workload into the stream of blended batches BlendServe runs
// (PAPER §4.4), each of which is one blended-batch attention step of this
// library.  Host only, integer arithmetic only (the memory partition is an exact rational
// computed with multi-limb integers), so results are bit-identical to oracle/sched.py.
//
//   1. scanner units: in preorder, a node whose children are all single-request leaves is
//      ONE merged unit (P:7 "merge sub-trees into single nodes if doing so does not hurt the
//      prefix sharing ratio"), every other node with ending requests is a unit of those;
//   2. two cursors walk the units from both ends, the memory M split into M_L, M_R
//      by  M_L + M_R = M,  M_L rho(R_L) + M_R rho(R_R) = M rho(rt) whenever a
//      cursor moves;
//   3. continuous batching per side with chunked prefill and a runtime
//      prefix cache of the active requests plus each side's last completed path.
// The readings of what §4.4 leaves open are DESIGN.md §3 #25-#31.
#include <algorithm>
#include <cstring>
#include <new>
#include <vector>

#include "blend.h"
#include "tree.h"

extern "C" int blend_internal_fail(int status, const char* msg);

struct blend_schedule {
  std::vector<int64_t> step_off{0};
  std::vector<int32_t> req, n_cached, q;
  std::vector<int32_t> order;
  std::vector<uint8_t> side;
  std::vector<int64_t> m_left;
  int64_t cached_prompt_tokens = 0, optimal_cached_tokens = 0;
};

namespace {

// Minimal unsigned multi-limb integer (32-bit limbs, little endian): products of 128-bit keys.
struct Big {
  std::vector<uint32_t> l;
  static Big of(u128 v) {
    Big b;
    while (v) {
      b.l.push_back((uint32_t)v);
      v >>= 32;
    }
    return b;
  }
  void trim() {
    while (!l.empty() && l.back() == 0) l.pop_back();
  }
};
Big mul(const Big& a, const Big& b) {
  Big r;
  if (a.l.empty() || b.l.empty()) return r;
  r.l.assign(a.l.size() + b.l.size(), 0);
  for (size_t i = 0; i < a.l.size(); ++i) {
    uint64_t carry = 0;
    for (size_t j = 0; j < b.l.size(); ++j) {
      uint64_t cur = (uint64_t)a.l[i] * b.l[j] + r.l[i + j] + carry;
      r.l[i + j] = (uint32_t)cur;
      carry = cur >> 32;
    }
    size_t k = i + b.l.size();
    while (carry) {
      uint64_t cur = (uint64_t)r.l[k] + carry;
      r.l[k++] = (uint32_t)cur;
      carry = cur >> 32;
    }
  }
  r.trim();
  return r;
}
int cmp(const Big& a, const Big& b) {
  if (a.l.size() != b.l.size()) return a.l.size() < b.l.size() ? -1 : 1;
  for (size_t i = a.l.size(); i-- > 0;)
    if (a.l[i] != b.l[i]) return a.l[i] < b.l[i] ? -1 : 1;
  return 0;
}
Big sub(const Big& a, const Big& b) {   // a >= b
  Big r = a;
  int64_t borrow = 0;
  for (size_t i = 0; i < r.l.size(); ++i) {
    int64_t cur = (int64_t)r.l[i] - (i < b.l.size() ? b.l[i] : 0) - borrow;
    borrow = cur < 0;
    r.l[i] = (uint32_t)(cur + (borrow << 32));
  }
  r.trim();
  return r;
}

// Step 3: M_L = floor(M (rho_rt - rho_R) / (rho_L - rho_R)) clamped to [0, M] when rho_L > rho_R,
// else M / 2; rho = CU / MU with MU = 0 meaning +infinity (oracle/sched.py partition).
int64_t partition(int64_t M, u128 cul, u128 mul_, u128 cur, u128 mur, u128 curt, u128 murt) {
  if (mur == 0) return M / 2;
  if (mul_ == 0) return murt == 0 ? M : 0;
  if (murt == 0) return M;
  const Big L1 = mul(Big::of(cul), Big::of(mur)), R1 = mul(Big::of(cur), Big::of(mul_));
  if (cmp(L1, R1) <= 0) return M / 2;                                // rho_L <= rho_R
  const Big T1 = mul(Big::of(curt), Big::of(mur)), T2 = mul(Big::of(cur), Big::of(murt));
  if (cmp(T1, T2) <= 0) return 0;                                    // rho_rt <= rho_R
  // ratio = (curt mur - cur murt) mul / ((cul mur - cur mul) murt) in (0, inf)
  const Big num = mul(sub(T1, T2), Big::of(mul_)), den = mul(sub(L1, R1), Big::of(murt));
  const Big Mnum = mul(Big::of((u128)M), num);
  if (cmp(mul(Big::of((u128)M), den), Mnum) <= 0) return M;           // ratio >= 1
  int64_t lo = 0, hi = M;                                             // largest x: x den <= M num
  while (lo < hi) {
    const int64_t mid = lo + (hi - lo + 1) / 2;
    if (cmp(mul(Big::of((u128)mid), den), Mnum) <= 0) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

struct Unit {
  int32_t node;
  std::vector<int32_t> reqs;
};

std::vector<Unit> scanner_units(const blend_tree* t) {
  const int32_t N = t->n_nodes;
  std::vector<std::vector<int32_t>> kids(N);
  for (int32_t i = 0; i < N; ++i)
    if (t->node_parent[i] >= 0) kids[t->node_parent[i]].push_back(i);
  auto nend = [&](int32_t x) { return t->node_end_off[x + 1] - t->node_end_off[x]; };
  std::vector<char> merged(N, 0), inside(N, 0);
  std::vector<Unit> units;
  for (int32_t x = 0; x < N; ++x) {
    const int32_t par = t->node_parent[x];
    if (par >= 0 && (inside[par] || merged[par])) {
      inside[x] = 1;
      continue;
    }
    bool all_single = !kids[x].empty();
    for (int32_t c : kids[x]) all_single = all_single && kids[c].empty() && nend(c) == 1;
    if (all_single || nend(x) > 0) {
      Unit u;
      u.node = x;
      for (int32_t k = t->node_end_off[x]; k < t->node_end_off[x + 1]; ++k) u.reqs.push_back(t->node_end_req[k]);
      if (all_single) {
        merged[x] = 1;
        for (int32_t c : kids[x]) u.reqs.push_back(t->node_end_req[t->node_end_off[c]]);
      }
      units.push_back(std::move(u));
    }
  }
  return units;
}

int32_t lcp(const blend_tree* t, int32_t a, int32_t b) {
  const int64_t a0 = t->req_path_off[a], a1 = t->req_path_off[a + 1];
  const int64_t b0 = t->req_path_off[b], b1 = t->req_path_off[b + 1];
  int32_t m = 0;
  for (int64_t i = 0; a0 + i < a1 && b0 + i < b1; ++i) {
    const int32_t x = t->req_path_nodes[a0 + i];
    if (x != t->req_path_nodes[b0 + i]) break;
    m = t->node_start[x] + t->node_len[x];
  }
  return m;
}

struct Active {
  int32_t r, side;
  int64_t mat, dec;   // materialised prompt tokens, decodes done
  int32_t prov;       // request providing the reused prompt prefix (-1: none)
  int64_t need;       // prefix length it must have materialised first
};

int schedule_impl(const blend_tree* t, const blend_sched_args* a, blend_schedule* S) {
  const int64_t M = a->mem_tokens;
  const int64_t chunk = a->chunk > 0 ? a->chunk : 512;
  const int64_t budget0 = a->step_budget > 0 ? a->step_budget : 8192;
  const bool dfs = a->policy == BLEND_SCHED_DFS;
  const int32_t R = t->n_req;
  const int32_t* p = t->prompt_len.data();
  const int32_t* d = t->out_len.data();
  std::vector<Unit> units;
  if (dfs) {
    Unit u;
    u.node = -1;
    u.reqs = t->dfs_order;
    units.push_back(std::move(u));
  } else {
    units = scanner_units(t);
  }
  u128 cu_rt = 0, mu_rt = 0;
  for (int32_t i = 0; i < t->n_nodes; ++i)
    if (t->node_parent[i] < 0) {
      cu_rt += t->cu[i];
      mu_rt += t->mu[i];
    }
  const int32_t K = (int32_t)units.size();
  int32_t L = 0, Rc = K - 1;
  bool met = K <= 1;
  // queues as (unit, position) cursors; `shared` is the unit both sides draw from once met
  int32_t qL = 0, qR = K > 1 ? K - 1 : -1, shared = 0;
  size_t pL = 0, pR = 0, pS = 0;
  int64_t m_left = M;
  auto repartition = [&]() {
    if (met) return;
    const int32_t xl = units[L].node, xr = units[Rc].node;
    m_left = partition(M, t->cu[xl], t->mu[xl], t->cu[xr], t->mu[xr], cu_rt, mu_rt);
  };
  repartition();
  int64_t used[2] = {0, 0};
  std::vector<Active> active;
  std::vector<int32_t> slot(R, -1);   // index of an active request in `active`, -1 otherwise
  int32_t last_done[2] = {-1, -1};    // each side's most recently completed request
  S->side.assign(R, 0);
  const int64_t max_steps = a->max_steps > 0 ? a->max_steps : INT64_MAX;
  for (int64_t step = 0; step < max_steps; ++step) {
    // ---- admission
    for (int s = 0; s < (dfs ? 1 : 2); ++s) {
      for (;;) {
        const Unit* qu;
        size_t* pos;
        if (met) {
          qu = &units[shared];
          pos = &pS;
        } else {
          qu = &units[s == 0 ? qL : qR];
          pos = s == 0 ? &pL : &pR;
        }
        if (*pos >= qu->reqs.size()) {
          if (met) break;
          if (s == 0 && L + 1 < Rc) {
            qL = ++L;
            pL = 0;
          } else if (s == 1 && Rc - 1 > L) {
            qR = --Rc;
            pR = 0;
          } else {   // the cursors meet on the other side's unit
            if (s == 0) {
              shared = qR;
              pS = pR;
            } else {
              shared = qL;
              pS = pL;
            }
            met = true;
          }
          repartition();
          continue;
        }
        const int64_t cap = s == 0 ? m_left : M - m_left;
        const int32_t r = qu->reqs[*pos];
        const int64_t fp = (int64_t)p[r] + d[r];
        if (used[s] > 0 && used[s] + fp > cap) break;
        ++*pos;
        // prefix sharing: reuse the longest prompt prefix shared with an active request or
        // with a side's most recently completed one (its path stays cached), capped at
        // that request's prompt; active requests in admission order first, ties to the first
        int64_t cached = 0;
        int32_t prov = -1;
        auto consider = [&](int32_t a2) {
          const int64_t c = std::min<int64_t>(lcp(t, r, a2), p[a2]);
          if (c > cached) {
            cached = c;
            prov = a2;
          }
        };
        for (const Active& e : active) consider(e.r);
        for (int sd = 0; sd < 2; ++sd)
          if (last_done[sd] >= 0) consider(last_done[sd]);
        cached = std::min<int64_t>(cached, std::max<int64_t>(0, (int64_t)p[r] - 1));
        S->cached_prompt_tokens += cached;
        used[s] += fp;
        active.push_back({r, s, cached, 0, cached > 0 ? prov : -1, cached});
        slot[r] = (int32_t)active.size() - 1;
        S->order.push_back(r);
        S->side[r] = (uint8_t)s;
      }
    }
    if (active.empty()) break;
    // ---- one step
    int64_t budget = budget0;
    for (Active& e : active) {
      if (e.mat < p[e.r]) {
        // wait until the provider (earlier in the batch) has materialised the reused prefix
        if (e.prov >= 0 && slot[e.prov] >= 0 && active[slot[e.prov]].mat < e.need) continue;
        const int64_t q = std::min<int64_t>(std::min<int64_t>(chunk, p[e.r] - e.mat), budget);
        if (q <= 0) continue;
        budget -= q;
        e.mat += q;
        S->req.push_back(e.r);
        S->n_cached.push_back((int32_t)e.mat);
        S->q.push_back((int32_t)q);
      } else {
        S->req.push_back(e.r);
        S->n_cached.push_back((int32_t)(p[e.r] + e.dec + 1));
        S->q.push_back(1);
        e.dec += 1;
      }
    }
    S->step_off.push_back((int64_t)S->req.size());
    S->m_left.push_back(m_left);
    size_t k = 0;
    for (const Active& e : active) {
      if (e.mat >= p[e.r] && e.dec >= d[e.r]) {
        used[e.side] -= (int64_t)p[e.r] + d[e.r];
        slot[e.r] = -1;
        last_done[e.side] = e.r;
      } else {
        slot[e.r] = (int32_t)k;
        active[k++] = e;
      }
    }
    active.resize(k);
  }
  // P:480's optimum: sum_r p_r - distinct prompt tokens of the tree (the c-2 clamp per node)
  std::vector<int64_t> maxp(t->n_nodes, 0);
  int64_t sum_p = 0;
  for (int32_t r = 0; r < R; ++r) {
    sum_p += p[r];
    for (int64_t k2 = t->req_path_off[r]; k2 < t->req_path_off[r + 1]; ++k2) {
      const int32_t x = t->req_path_nodes[k2];
      maxp[x] = std::max<int64_t>(maxp[x], p[r]);
    }
  }
  int64_t distinct = 0;
  for (int32_t x = 0; x < t->n_nodes; ++x)
    distinct += std::max<int64_t>(0, std::min<int64_t>(maxp[x] - t->node_start[x], t->node_len[x]));
  S->optimal_cached_tokens = sum_p - distinct;
  return BLEND_OK;
}

}  // namespace

extern "C" {

int blend_schedule_build(const blend_tree* t, const blend_sched_args* a, blend_schedule** out) {
  if (!t || !a || !out) return blend_internal_fail(BLEND_EINVAL, "schedule: NULL argument");
  *out = nullptr;
  if (a->mem_tokens <= 0 || a->chunk < 0 || a->step_budget < 0 || a->max_steps < 0 ||
      (a->policy != BLEND_SCHED_DUAL && a->policy != BLEND_SCHED_DFS))
    return blend_internal_fail(BLEND_EINVAL, "schedule: mem_tokens / chunk / step_budget / max_steps / policy");
  blend_schedule* S = new (std::nothrow) blend_schedule();
  if (!S) return blend_internal_fail(BLEND_ENOMEM, "out of host memory");
  int st;
  try {
    st = schedule_impl(t, a, S);
  } catch (const std::bad_alloc&) {
    st = blend_internal_fail(BLEND_ENOMEM, "out of host memory");
  }
  if (st) {
    delete S;
    return st;
  }
  *out = S;
  return BLEND_OK;
}

int blend_schedule_get_view(const blend_schedule* S, blend_schedule_view* v) {
  if (!S || !v) return blend_internal_fail(BLEND_EINVAL, "schedule view: NULL argument");
  v->n_steps = (int64_t)S->m_left.size();
  v->n_entries = (int64_t)S->req.size();
  v->n_req = (int32_t)S->side.size();
  v->step_off = S->step_off.data();
  v->req = S->req.data();
  v->n_cached = S->n_cached.data();
  v->q = S->q.data();
  v->order = S->order.data();
  v->n_admitted = (int32_t)S->order.size();
  v->side = S->side.data();
  v->m_left = S->m_left.data();
  v->cached_prompt_tokens = S->cached_prompt_tokens;
  v->optimal_cached_tokens = S->optimal_cached_tokens;
  return BLEND_OK;
}

void blend_schedule_free(blend_schedule* S) { delete S; }

}  // extern "C"
