// tree.h — the host-side descriptor tree (opaque blend_tree of include/blend.h), shared by
// the builder / planner / sharder (host.cpp) and the batch former (sched.cpp).
// Not part of the public ABI.
#pragma once
#include <stdint.h>

#include <vector>

#include "blend.h"

using u128 = unsigned __int128;
using i128 = __int128;

struct blend_tree {
  // ---- owned inputs
  blend_build_args args{};
  std::vector<int64_t> tok_off;
  std::vector<int32_t> tokens, q_len, prompt_len, out_len, free_pages;
  std::vector<int64_t> global_id;
  std::vector<int32_t> req_group;   // Alg. 2 relocation group per request (0: not relocated)
  bool has_free = false;
  int32_t rows_min = 128, min_sep_len = 128, force_class = 0;
  // ---- descriptors
  int32_t n_req = 0, n_nodes = 0;
  std::vector<int32_t> node_parent, node_start, node_len, node_first_req, node_nreq;
  std::vector<int64_t> node_page_off;
  std::vector<uint8_t> node_class;
  std::vector<uint64_t> node_key_cu, node_key_mu;
  std::vector<u128> cu, mu;
  std::vector<int32_t> node_end_off, node_end_req;   // requests ending at each node (ascending)
  std::vector<int32_t> page_table;
  std::vector<int64_t> req_path_off;
  std::vector<int32_t> req_path_nodes;
  std::vector<int64_t> req_q_off;
  std::vector<uint8_t> req_class;
  std::vector<int32_t> req_dfs_rank, dfs_order;
  // ---- plan (host image of the device plan buffer)
  std::vector<uint8_t> plan_blob;
  int64_t sec_off[16] = {0}, sec_count[16] = {0};
  blend_plan_info info{};
  size_t workspace_bytes = 0;
  int64_t n_partial_rows = 0;
  int64_t stream_entries = 0;   // sum over stream units of their entry counts (launch heuristic)
  int32_t dense_ctas = 0;       // dense-pass grid cap (0: one CTA per SM), set by the planner
  int32_t merge_nsrc = 0;       // > 0: every merge list has this many sources
  int32_t max_page = -1;        // largest physical page id in page_table (-1: no pages)
};
