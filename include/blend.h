/*
 * blend.h — C ABI of libblend: blended-batch attention over a radix-tree paged
 * KV cache, the data-parallel hot path of BlendServe (arXiv 2411.16102).
 *
 * Citations: "P:n" = PAPER.md line n (the paper's LaTeX source), "§x" = its
 * section.  The operation the library computes is exact causal GQA attention
 * (reading #1-#3 in DESIGN.md) for every query token of a batch whose
 * requests' cached token paths form a prefix tree:
 *   - the tree is the paper's Trie (§4.1: "each leaf node ...
 *     represents an actual request while each internal node is a segment of
 *     the prefix shared by all its descendants");
 *   - nodes are ordered by compute density rho = Comp/Mem (§2.3 P:87-96,
 *     §4.2) with the layer-wise sort of Algorithm 1 (§4.3);
 *   - a shared prefix node is attended ONCE for all the requests under it
 *     ("exactly-once computation of shared prefixes for a single batch", §5
 *     P:11; the cascade variant "reusing the KV-cache access shared by the
 *     common prefix", §7.2), each request's private suffix
 *     separately, and the partial results are merged by log-sum-exp;
 *   - the tree is split across data-parallel GPUs "from both sides" (§7.1
 *     P:246) by blend_shard.
 *
 * Conventions (all functions):
 *   - return BLEND_OK (0) or a negative blend_status, never throw, never abort;
 *     blend_last_error() gives a thread-local message for the last failure;
 *   - "host" pointers are CPU memory, "device" pointers are CUDA global memory
 *     of the current device; streams and events are passed as void* and are
 *     cudaStream_t / cudaEvent_t;
 *   - the library never allocates device memory and never synchronises a
 *     stream: the caller owns q, caches, out, lse, plan buffer and workspace.
 */
#ifndef BLEND_H
#define BLEND_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BLEND_ABI_VERSION 2

typedef enum {
  BLEND_OK = 0,
  BLEND_EINVAL = -1,       /* invalid dims / dtype / flags / NULL argument / duplicate page ids */
  BLEND_EMALFORMED = -2,   /* malformed tree input: empty path, q_len out of range, negative token */
  BLEND_ENOSPC = -3,       /* too few free pages, or buffer / workspace too small */
  BLEND_ECUDA = -4,        /* a CUDA launch or runtime call failed (cudaPeekAtLastError) */
  BLEND_ENOMEM = -5,       /* host allocation failed */
  BLEND_EUNSUPPORTED = -6  /* head_dim not in {64,128}, or device is not sm_100 */
} blend_status;

enum { BLEND_BF16 = 0, BLEND_F32 = 1 };

/* thread-local message of the last failing blend_* call on this thread */
const char* blend_last_error(void);
int blend_abi_version(void);

/* ------------------------------------------------------------------------ */
/* Descriptor builder (host only).                                           */
/* ------------------------------------------------------------------------ */
typedef struct {
  int32_t n_req;               /* R >= 1 requests of this batch                                  */
  const int64_t* tok_off;      /* host [R+1] CSR offsets into tokens                             */
  const int32_t* tokens;       /* host: request r's cached token path tokens[tok_off[r]..tok_off[r+1]),
                                  ids >= 0; its LAST q_len[r] tokens are this step's queries and
                                  their K/V are already in the cache (reading #3)               */
  const int32_t* q_len;        /* host [R], 1 <= q_len[r] <= path length                         */
  const int32_t* prompt_len;   /* host [R] p_r >= 0 (density only)                         */
  const int32_t* out_len;      /* host [R] d_r >= 0, estimated output length (density only)     */
  const int64_t* global_id;    /* host [R] global request index, or NULL = 0..R-1                */
  int32_t num_q_heads;         /* Hq, multiple of num_kv_heads (GQA, kvh = h / (Hq/Hkv))        */
  int32_t num_kv_heads;        /* Hkv                                                            */
  int32_t head_dim;            /* D in {64, 128}                                                 */
  int32_t kv_dtype;            /* BLEND_BF16 | BLEND_F32 (q/out use the same dtype)              */
  int64_t model_params;        /* P_model, e.g. 8030261248 for Llama-3.1-8B              */
  int32_t hidden;              /* H                                                       */
  int32_t layers;              /* L                                                       */
  int32_t page_size;           /* ps: power of two in [16, 128]                                  */
  const int32_t* free_pages;   /* host [n_free_pages] physical page ids handed out in node-id
                                  order, or NULL = 0,1,2,...; used ids must be distinct, >= 0    */
  int64_t n_free_pages;
  int32_t rows_min;            /* SMALL/BIG and SEPARATE row threshold, 0 = default 128   */
  int32_t min_sep_len;         /* SEPARATE needs len >= this, -1 = default 128, 0 = off  */
  int32_t force_class;         /* 0 auto | 1 every shared node SEPARATE for all its requests
                                  ("literal cascade") | 2 no node SEPARATE (all folded)        */
  int32_t split_tokens;        /* streaming split-KV chunk in tokens, 0 = auto (plan only)       */
  int32_t num_sms;             /* SM count the plan is sized for, 0 = 148 (B200)                */
  int32_t dense_split;         /* split-KV factor of dense items, 0 = auto (plan only)            */
  int32_t split_waste;         /* Alg. 2 conditional node splitting threshold t in
                                  tokens: an outlier subtree (density on the other side of the
                                  root density than its siblings') is relocated to the top level,
                                  duplicating its shared prefix, iff that prefix is <= t tokens.
                                  0 = off                                                        */
} blend_build_args;

typedef struct blend_tree blend_tree;   /* opaque, host-owned */

/* Read-only arrays owned by the tree (valid until blend_tree_free).  Node ids
 * are the preorder index of the density-sorted forest (Alg. 1, reading #11);
 * every node starts on a fresh page (reading #19). */
typedef struct {
  int32_t n_req, n_nodes;
  int64_t n_pages;                 /* = node_page_off[n_nodes]                              */
  const int32_t* node_parent;      /* [n_nodes] parent id, -1 for a top-level node          */
  const int32_t* node_start;       /* [n_nodes] absolute position of the node's first token */
  const int32_t* node_len;         /* [n_nodes] tokens in the node                          */
  const int64_t* node_page_off;    /* [n_nodes+1] CSR into page_table                       */
  const uint8_t* node_class;       /* [n_nodes] 1 = SEPARATE (attended once for its SMALL
                                      requests), 0 = folded into each request's own item   */
  const uint64_t* node_key_cu;     /* [n_nodes][2] (lo, hi) of the 128-bit compute key CU   */
  const uint64_t* node_key_mu;     /* [n_nodes][2] (lo, hi) of the 128-bit memory key MU    */
  const int32_t* node_first_req;   /* [n_nodes] smallest request id through the node        */
  const int32_t* node_nreq;        /* [n_nodes] |A(N)|, requests through the node           */
  const int32_t* page_table;       /* [n_pages] physical page ids                           */
  const int64_t* req_path_off;     /* [R+1] CSR into req_path_nodes                         */
  const int32_t* req_path_nodes;   /* root->end node ids of each request                    */
  const int64_t* req_q_off;        /* [R+1] query-row offsets (caller request order)        */
  const uint8_t* req_class;        /* [R] 1 = BIG (q_len*g >= rows_min), 0 = SMALL          */
  const int32_t* req_dfs_rank;     /* [R] position of the request in the DFS order          */
  const int64_t* req_global_id;    /* [R] global request index                              */
  const int32_t* req_group;        /* [R] Alg. 2 relocation group (0 = not relocated)        */
} blend_tree_view;

/* Build the descriptors for one batch.  Errors: EINVAL (dims, flags, NULLs,
 * duplicate or negative page ids), EUNSUPPORTED (head_dim), EMALFORMED (paths,
 * q_len, tokens), ENOSPC (free list too short), ENOMEM.  Deterministic: equal
 * inputs give byte-equal descriptors.  Reentrant (no globals). */
int blend_tree_build(const blend_build_args* args, blend_tree** out);
int blend_tree_get_view(const blend_tree* tree, blend_tree_view* view);
void blend_tree_free(blend_tree* tree);

/* Golden text dump (SPEC S:238 style), one line per node in id order:
 *   <2*depth spaces>#id start=S len=L tok=[<=8 ids] cu=CU mu=MU cls=S|F nreq=N ends=[ids]
 * Writes at most cap bytes (NUL-terminated if cap > 0); *need = bytes required
 * including the NUL.  ENOSPC if cap < *need. */
int blend_tree_dump(const blend_tree* tree, char* buf, size_t cap, size_t* need);

/* ------------------------------------------------------------------------ */
/* Data-parallel sharder (host only), §7.1 P:246.                             */
/* ------------------------------------------------------------------------ */
/* Splits the request DFS order into 2G weight-balanced blocks (weight =
 * 4*D*Hq*sum(pos+1) + kappa * first-touch KV bytes), cuts snapped to subtree
 * boundaries, shard g = block g + block 2G-1-g.  req_shard: host [n_req] out.
 * shards: host [n_shards] out, each a tree of the shard's requests in
 * ascending global id order built with the parent's build args and
 * shard_free_pages[g] (NULL entries / NULL array = 0,1,2,...).  An empty
 * shard yields shards[g] = NULL.  Caller frees every non-NULL shard tree.
 * kappa <= 0 selects 213 (measured B200 ridge, FLOP/byte). */
int blend_shard(const blend_tree* tree, int32_t n_shards, int64_t kappa,
                const int32_t* const* shard_free_pages, const int64_t* n_shard_free,
                int32_t* req_shard, blend_tree** shards);

/* ------------------------------------------------------------------------ */
/* Dual-scanner batch former (host only), NEXT-2: PAPER §4.4 P:354-380.        */
/* ------------------------------------------------------------------------ */
/* The tree is a whole offline workload: each request's path is its full PROMPT
 * (prompt_len = path length) and out_len its output length d.  The former walks the
 * density-sorted tree's scanner units (a node whose children are all single-request
 * leaves is one merged unit, P:7) from both ends with two cursors, splits the KV memory
 * M into M_L + M_R = M with M_L rho(R_L) + M_R rho(R_R) = M rho(rt) whenever a cursor
 * moves (exact integer arithmetic, floor), admits requests per side while
 * their footprint p + d fits (continuous batching), reuses the prompt prefix an
 * active request already materialised (runtime prefix cache), and emits one blended
 * batch per step: chunked prefill (<= chunk tokens per request, <= step_budget per step)
 * then d decode steps.  Deterministic; readings in DESIGN.md §3 #25-#31. */
enum { BLEND_SCHED_DUAL = 0, BLEND_SCHED_DFS = 1 };

typedef struct {
  int64_t mem_tokens;     /* M: KV memory in tokens (all layers), > 0                      */
  int32_t chunk;          /* chunked-prefill tokens per request per step, 0 = 512           */
  int32_t step_budget;    /* prefill tokens per step, 0 = 8192                              */
  int32_t policy;         /* BLEND_SCHED_DUAL, or BLEND_SCHED_DFS: the tree's DFS order on one
                             side with all of M (the sharing reference)              */
  int64_t max_steps;      /* stop after this many steps, 0 = run to completion              */
} blend_sched_args;

typedef struct blend_schedule blend_schedule;   /* opaque, host-owned */

/* Read-only arrays owned by the schedule (valid until blend_schedule_free). */
typedef struct {
  int64_t n_steps, n_entries;
  int32_t n_req, n_admitted;
  const int64_t* step_off;     /* [n_steps+1] CSR of the steps' batch entries            */
  const int32_t* req;          /* [n_entries] tree request index                         */
  const int32_t* n_cached;     /* [n_entries] the request's cached path length after the step
                                  (prompt[:n] while prefilling; prompt + n - p generated
                                  tokens while decoding): the step batch's path length   */
  const int32_t* q;            /* [n_entries] the step's query tokens (last q of the path) */
  const int32_t* order;        /* [n_admitted] requests in admission order               */
  const uint8_t* side;         /* [n_req] 0 = left (compute-intensive), 1 = right cursor  */
  const int64_t* m_left;       /* [n_steps] M_L in force during the step                 */
  int64_t cached_prompt_tokens;   /* prompt tokens reused from the runtime cache           */
  int64_t optimal_cached_tokens;  /* sum p - distinct prompt tokens (P:480's optimum)       */
} blend_schedule_view;

/* EINVAL (NULLs, mem_tokens <= 0, negative chunk / budget / max_steps, bad policy),
 * ENOMEM.  Reentrant. */
int blend_schedule_build(const blend_tree* tree, const blend_sched_args* args, blend_schedule** out);
int blend_schedule_get_view(const blend_schedule* sched, blend_schedule_view* view);
void blend_schedule_free(blend_schedule* sched);

/* ------------------------------------------------------------------------ */
/* Work plan + attention (device).                                            */
/* ------------------------------------------------------------------------ */
typedef struct {
  int64_t n_tokens;          /* sum q_len = rows of q/out                         */
  int64_t n_items;           /* SEPARATE-node items + request items               */
  int64_t n_dense_units;     /* tensor-core (tcgen05) work units                  */
  int64_t n_stream_units;    /* HBM-streaming work units                          */
  int64_t n_partial_rows;    /* partial (o, lse) rows in the workspace            */
  int64_t n_merge_tokens;    /* query tokens with >= 2 partial sources            */
  int64_t n_entries;         /* KV page entries referenced by the plan            */
  int64_t dense_kv_tokens;   /* sum over dense units of KV tokens read (per kvh)  */
  int64_t stream_kv_tokens;  /* sum over stream units of KV tokens read (per kvh) */
} blend_plan_info;

int blend_plan_get_info(const blend_tree* tree, blend_plan_info* info);

/* Bytes of the device plan buffer / of the attention workspace. */
size_t blend_plan_bytes(const blend_tree* tree);
size_t blend_workspace_bytes(const blend_tree* tree);

/* Uploaded plan: the caller's plan buffer plus the planner's scalars.  Filled by
 * blend_plan_upload; read-only for the caller (blend_attention trusts it). */
typedef struct {
  const void* dev;           /* caller device buffer holding the plan                        */
  size_t bytes;
  int64_t off[16];           /* byte offset of each plan section inside dev (library layout) */
  int64_t count[16];         /* element count of each plan section                          */
  int32_t num_q_heads, num_kv_heads, head_dim, kv_dtype, page_size;   /* the tree's build args */
  int32_t dense_ctas;        /* dense-pass grid cap for the overlapped launch (planner's SM
                                share for NEXT-1); 0 = one CTA per SM              */
  int64_t n_partial_rows;    /* partial (o, lse) rows the workspace holds                    */
  int64_t stream_entries;    /* sum of KV entries over the streaming units (launch sizing)   */
  int32_t merge_nsrc;        /* > 0: every merge list has exactly this many partial rows     */
  int32_t max_page;          /* largest physical page id the plan reads (-1: none);
                                blend_attention requires max_page < n_cache_pages           */
} blend_plan;

/* Copy the plan (host, inside the tree) into dev_buf (device, >= blend_plan_bytes)
 * with cudaMemcpyAsync on stream.  The tree may be freed after the copy has
 * completed; the plan struct stays valid as long as dev_buf does.  ENOSPC if
 * bytes is too small, ECUDA on copy failure. */
int blend_plan_upload(const blend_tree* tree, void* dev_buf, size_t bytes, void* stream,
                      blend_plan* plan);

enum { BLEND_PATH_AUTO = 0, BLEND_PATH_GENERIC = 1, BLEND_PATH_NO_TCGEN05 = 2 };
enum { BLEND_SERIALIZE = 1 };

typedef struct {
  const void* q;             /* device [sum q, Hq, D] (kv dtype), rows in caller request order:
                                request r owns rows req_q_off[r].., positions n_r-q_r..n_r-1 */
  const void* k_cache;       /* device [n_cache_pages, Hkv, ps, D]: each (page, kv head) block is
                                one contiguous ps*D run (head-major within a page)            */
  const void* v_cache;       /* device, same layout as k_cache                               */
  int64_t n_cache_pages;     /* pages in the cache allocations (page ids must be < this)     */
  void* out;                 /* device [sum q, Hq, D] (kv dtype), written                    */
  float* lse;                /* device [sum q, Hq] fp32 natural-log LSE, written             */
  void* workspace;           /* device, >= blend_workspace_bytes (always required): partial
                                (o, lse) rows and the streaming pass's unit counter (reset by
                                every call); scratch between calls.  One call in flight per
                                workspace                                                   */
  size_t workspace_bytes;
  const blend_plan* plan;    /* from blend_plan_upload (its buffer must be resident)         */
  int32_t dtype;             /* BLEND_BF16 | BLEND_F32: element type of q, k/v caches and out;
                                must equal the plan's kv_dtype (EINVAL otherwise)           */
  int32_t path;              /* BLEND_PATH_*: AUTO = tcgen05 dense + streaming (+ generic for
                                fp32); GENERIC = every unit on the fp32-FMA item executor;
                                NO_TCGEN05 = dense units on the generic executor            */
  int32_t flags;             /* BLEND_SERIALIZE: run the passes back to back.  Default: the
                                streaming pass is launched with programmatic dependent launch
                                and overlaps the dense pass on free SMs (the two passes are
                                independent; the streaming grid completes only after the
                                dense grid) and the merge kernel is a programmatic
                                dependent of the streaming grid                            */
  void* events[4];           /* optional cudaEvent_t recorded before dense, before stream,
                                before merge, after merge (NULL entries skipped); non-NULL
                                events[1] or events[2] imply BLEND_SERIALIZE                 */
} blend_attn_args;

/* Enqueue the blended-batch attention on stream.  The slots of a node's pages that
 * hold its tokens must be finite; the slots past a node's end (the tail of its last
 * page) may hold anything, NaN included: the kernels never let them reach the output.
 * Never allocates, never synchronises; asynchronous faults surface at the caller's
 * next synchronisation.  EINVAL (NULLs, dtype != plan kv_dtype, a plan page id
 * >= n_cache_pages, bad path / flags), ENOSPC (workspace), EUNSUPPORTED (not sm_100),
 * ECUDA (launch failure). */
int blend_attention(const blend_attn_args* args, void* stream);

/* ------------------------------------------------------------------------ */
/* Synthetic input fillers (bench / tests; SURVEY.md §8(c-7) generator).      */
/* ------------------------------------------------------------------------ */
/* K/V cache fill: for i < n_pages, page page_ids[i] slot s < page_count[i] gets, for the
 * cache's kv head k < num_kv_heads (global kv head kvh = kv_head0 + k: a head-parallel
 * rank's slice keeps the full problem's values),
 * KV[k][e] = grid(mix(page_hash[i*ps+s] ^ mix(seed_kv + ((kind*2^8 + kvh)*2^12 + e))))
 * with seed_kv = seed ^ 0x5BD1E9955BD1E995; slots >= page_count[i] are zeroed.
 * page_ids, page_count, page_hash are DEVICE arrays. */
int blend_fill_kv(void* k_cache, void* v_cache, int32_t kv_dtype, int32_t num_kv_heads,
                  int32_t kv_head0, int32_t head_dim, int32_t page_size, const int32_t* page_ids,
                  const int32_t* page_count, const uint64_t* page_hash, int64_t n_pages,
                  uint64_t seed, void* stream);

/* Q fill: row i, q head k < num_q_heads (global head h = head0 + k) gets
 * Q[k][e] = scale_q * grid(mix(seed_q ^ mix(((gid*2^20 + t)*2^8 + h)*2^12 + e)))
 * (all arithmetic mod 2^64; kind 0 = K, 1 = V; grid(z) = ((z>>56) - 128) / 128)
 * with gid = row_gid[i], t = row_t[i], seed_q = seed ^ 0xC2B2AE3D27D4EB4F.  DEVICE arrays. */
int blend_fill_q(void* q, int32_t dtype, int32_t num_q_heads, int32_t head0, int32_t head_dim,
                 const int64_t* row_gid, const int32_t* row_t, int64_t n_rows, uint64_t seed,
                 float scale_q, void* stream);

/* Write `bytes` of a device scratch buffer (L2 flush between timed steps). */
int blend_l2_flush(void* buf, size_t bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* BLEND_H */
