// attention.cu — blend_plan_upload and blend_attention: validates arguments and
// enqueues the dense pass (tcgen05), the streaming pass and the LSE merge on the
// caller's stream.  Never allocates, never synchronises.
#include <cuda_runtime.h>
#include <math.h>

#include "blend.h"
#include "common.cuh"

extern "C" int blend_internal_fail(int status, const char* msg);
extern "C" int blend_internal_plan_image(const blend_tree* t, const void** data, size_t* bytes, const int64_t** off,
                                         const int64_t** count);
extern "C" int blend_internal_tree_dims(const blend_tree* t, int32_t* dims);
extern "C" int64_t blend_internal_partial_rows(const blend_tree* t);
extern "C" int64_t blend_internal_stream_entries(const blend_tree* t);
extern "C" int32_t blend_internal_merge_nsrc(const blend_tree* t);
extern "C" int32_t blend_internal_dense_ctas(const blend_tree* t);
extern "C" int32_t blend_internal_max_page(const blend_tree* t);

namespace blend {
cudaError_t launch_generic(const AttnParams& p, cudaStream_t st);
cudaError_t launch_merge(const AttnParams& p, cudaStream_t st, bool pdl);
cudaError_t launch_streamw(const AttnParams& p, int64_t n_cache_pages, cudaStream_t st, bool overlap);
cudaError_t launch_dense(const AttnParams& p, int64_t n_cache_pages, cudaStream_t st);
cudaError_t launch_dense_ks(const AttnParams& p, int64_t n_cache_pages, cudaStream_t st, bool overlap);
}  // namespace blend

// Diagnostics (blend_internal_set_trace / _set_stats): per-thread so that callers
// driving several devices from several threads do not share them.
static thread_local unsigned long long* g_trace = nullptr;   // timeline stamps
static thread_local unsigned long long* g_stats = nullptr;   // softmax path counters
extern "C" int blend_internal_set_trace(void* dev) {
  g_trace = (unsigned long long*)dev;
  return 0;
}
extern "C" int blend_internal_set_stats(void* dev) {
  g_stats = (unsigned long long*)dev;
  return 0;
}

namespace {
int cuda_fail(cudaError_t e) { return blend_internal_fail(BLEND_ECUDA, cudaGetErrorString(e)); }

int check_arch() {
  int dev = 0, major = 0, minor = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return cuda_fail(cudaGetLastError());
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  if (major != 10 || minor != 0) return blend_internal_fail(BLEND_EUNSUPPORTED, "libblend is built for sm_100a (B200)");
  return BLEND_OK;
}
}  // namespace

extern "C" int blend_plan_upload(const blend_tree* tree, void* dev_buf, size_t bytes, void* stream, blend_plan* plan) {
  if (!tree || !dev_buf || !plan) return blend_internal_fail(BLEND_EINVAL, "plan_upload: NULL argument");
  const void* data;
  size_t need;
  const int64_t *off, *count;
  int st = blend_internal_plan_image(tree, &data, &need, &off, &count);
  if (st) return st;
  if (bytes < need) return blend_internal_fail(BLEND_ENOSPC, "plan_upload: buffer too small");
  cudaError_t e = cudaMemcpyAsync(dev_buf, data, need, cudaMemcpyHostToDevice, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e);
  plan->dev = dev_buf;
  plan->bytes = need;
  for (int i = 0; i < 16; ++i) {
    plan->off[i] = off[i];
    plan->count[i] = count[i];
  }
  int32_t dims[5];
  blend_internal_tree_dims(tree, dims);
  plan->num_q_heads = dims[0];
  plan->num_kv_heads = dims[1];
  plan->head_dim = dims[2];
  plan->kv_dtype = dims[3];
  plan->page_size = dims[4];
  plan->dense_ctas = blend_internal_dense_ctas(tree);
  plan->n_partial_rows = blend_internal_partial_rows(tree);
  plan->stream_entries = blend_internal_stream_entries(tree);
  plan->merge_nsrc = blend_internal_merge_nsrc(tree);
  plan->max_page = blend_internal_max_page(tree);
  return BLEND_OK;
}

extern "C" int blend_attention(const blend_attn_args* a, void* stream) {
  using namespace blend;
  if (!a || !a->plan || !a->q || !a->k_cache || !a->v_cache || !a->out || !a->lse)
    return blend_internal_fail(BLEND_EINVAL, "attention: NULL argument");
  const blend_plan& pl = *a->plan;
  if (!pl.dev) return blend_internal_fail(BLEND_EINVAL, "attention: plan not uploaded");
  if (a->path < 0 || a->path > 2) return blend_internal_fail(BLEND_EINVAL, "attention: bad path");
  if (a->flags & ~BLEND_SERIALIZE) return blend_internal_fail(BLEND_EINVAL, "attention: bad flags");
  if (a->dtype != pl.kv_dtype) return blend_internal_fail(BLEND_EINVAL, "attention: dtype differs from the plan's kv_dtype");
  if (a->n_cache_pages <= 0 || pl.max_page >= a->n_cache_pages)
    return blend_internal_fail(BLEND_EINVAL, "attention: the plan reads a page id >= n_cache_pages");
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return cuda_fail(cudaGetLastError());
  static int arch_ok[64];   // per device: 0 unknown, 1 sm_100, -1 other
  if (dev < 64 && arch_ok[dev] == 0) arch_ok[dev] = check_arch() == BLEND_OK ? 1 : -1;
  if (dev >= 64 ? check_arch() != BLEND_OK : arch_ok[dev] < 0)
    return blend_internal_fail(BLEND_EUNSUPPORTED, "libblend is built for sm_100a (B200)");
  const int64_t prow = pl.n_partial_rows;
  const int hq = pl.num_q_heads, D = pl.head_dim;
  const size_t o_bytes = ((size_t)prow * hq * D * 4 + 255) & ~size_t(255);
  const size_t lse_bytes = ((size_t)prow * hq * 4 + 255) & ~size_t(255);
  const size_t need = o_bytes + lse_bytes + 256;   // + the streaming pass's unit counter
  if (!a->workspace || a->workspace_bytes < need)
    return blend_internal_fail(BLEND_ENOSPC, "attention: workspace too small");

  const char* base = (const char*)pl.dev;
  AttnParams p{};
  p.q = a->q;
  p.k_cache = a->k_cache;
  p.v_cache = a->v_cache;
  p.out = a->out;
  p.lse = a->lse;
  p.ws_o = (float*)a->workspace;
  p.ws_lse = (float*)((char*)a->workspace + o_bytes);
  p.sched = (int32_t*)((char*)a->workspace + o_bytes + lse_bytes);
  p.tok_pos = (const int32_t*)(base + pl.off[SEC_TOK_POS]);
  p.item_tokens = (const int32_t*)(base + pl.off[SEC_ITEM_TOKENS]);
  p.entries = (const KvEntry*)(base + pl.off[SEC_ENTRIES]);
  p.partmap = (const int32_t*)(base + pl.off[SEC_PARTMAP]);
  p.merge_tok = (const int32_t*)(base + pl.off[SEC_MERGE_TOK]);
  p.merge_off = (const int32_t*)(base + pl.off[SEC_MERGE_OFF]);
  p.srows = (const RowDesc*)(base + pl.off[SEC_STREAM_ROWS]);
  p.dqtok = (const int32_t*)(base + pl.off[SEC_DENSE_QTOK]);
  p.n_tokens = (int32_t)pl.count[SEC_TOK_POS];
  p.n_merge = (int32_t)pl.count[SEC_MERGE_TOK];
  p.hq = hq;
  p.hkv = pl.num_kv_heads;
  p.g = hq / pl.num_kv_heads;
  p.d = D;
  p.ps = pl.page_size;
  p.kv_f32 = pl.kv_dtype == BLEND_F32;
  p.scale_log2 = kLog2e / sqrtf((float)D);
  p.stats = g_stats;
  cudaStream_t st = (cudaStream_t)stream;
  const bool generic = a->path == BLEND_PATH_GENERIC || p.kv_f32;
  // PDL overlap of the independent dense and streaming passes, unless serialisation is
  // requested or per-pass events are wanted
  const bool overlap = !generic && !(a->flags & BLEND_SERIALIZE) && !a->events[1] && !a->events[2];
  cudaError_t e;

  if (a->events[0]) cudaEventRecord((cudaEvent_t)a->events[0], st);
  AttnParams pd = p;
  pd.units = (const Unit*)(base + pl.off[SEC_DENSE_UNITS]);
  pd.n_units = (int32_t)pl.count[SEC_DENSE_UNITS];
  // The streaming pass hands out units through a counter in the workspace.  The tcgen05
  // dense kernel zeroes it before its launch trigger (so the overlapped streaming grid
  // sees 0); without that kernel a memset ahead of the passes does.
  const bool stream_dyn = !generic && pl.count[SEC_STREAM_UNITS] > 0;
  const bool dense_tc = !generic && a->path != BLEND_PATH_NO_TCGEN05 && pd.n_units > 0;
  pd.trace = g_trace;
  pd.dense_ctas = overlap ? pl.dense_ctas : 0;   // the cap only makes room for the overlapped streaming grid
  pd.sched = stream_dyn && dense_tc ? p.sched : nullptr;
  if (stream_dyn && !dense_tc) {
    e = cudaMemsetAsync(p.sched, 0, sizeof(int32_t), st);
    if (e != cudaSuccess) return cuda_fail(e);
  }
  if (generic || a->path == BLEND_PATH_NO_TCGEN05) e = launch_generic(pd, st);
  else e = launch_dense(pd, a->n_cache_pages, st);
  if (e != cudaSuccess) return cuda_fail(e);
  // key-split units (<= 128 rows): dense_ks.cu, after the two-tile grid when serialised,
  // after the streaming grid (its PDL dependent) when overlapped; generic paths run them
  // with the other units
  AttnParams pk = p;
  pk.units = (const Unit*)(base + pl.off[SEC_DENSE_KS]);
  pk.n_units = (int32_t)pl.count[SEC_DENSE_KS];
  pk.dqtok = (const int32_t*)(base + pl.off[SEC_DENSE_KS_QTOK]);
  pk.trace = nullptr;
  pk.sched = nullptr;
  const bool ks_tc = pk.n_units > 0 && !generic && a->path != BLEND_PATH_NO_TCGEN05;
  if (pk.n_units > 0 && !ks_tc) {
    e = launch_generic(pk, st);
    if (e != cudaSuccess) return cuda_fail(e);
  }
  if (ks_tc && !overlap) {
    e = launch_dense_ks(pk, a->n_cache_pages, st, false);
    if (e != cudaSuccess) return cuda_fail(e);
  }

  if (a->events[1]) cudaEventRecord((cudaEvent_t)a->events[1], st);
  AttnParams ps_ = p;
  ps_.units = (const Unit*)(base + pl.off[SEC_STREAM_UNITS]);
  ps_.n_units = (int32_t)pl.count[SEC_STREAM_UNITS];
  ps_.avg_entries = ps_.n_units > 0 ? (int32_t)(pl.stream_entries / ps_.n_units) : 0;
  ps_.trace = g_trace;
  if (generic) e = launch_generic(ps_, st);
  else e = launch_streamw(ps_, a->n_cache_pages, st, overlap);
  if (e != cudaSuccess) return cuda_fail(e);
  if (ks_tc && overlap) {
    e = launch_dense_ks(pk, a->n_cache_pages, st, true);
    if (e != cudaSuccess) return cuda_fail(e);
  }

  if (a->events[2]) cudaEventRecord((cudaEvent_t)a->events[2], st);
  AttnParams pm = p;
  pm.trace = g_trace;
  pm.merge_nsrc = pl.merge_nsrc;
  e = launch_merge(pm, st, overlap);
  if (e != cudaSuccess) return cuda_fail(e);
  if (a->events[3]) cudaEventRecord((cudaEvent_t)a->events[3], st);
  e = cudaPeekAtLastError();
  if (e != cudaSuccess) return cuda_fail(e);
  return BLEND_OK;
}
