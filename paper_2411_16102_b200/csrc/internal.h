// internal.h — layouts shared by the host planner (host.cpp) and the kernels (*.cu).
// Not part of the public ABI (include/blend.h).
#pragma once
#include <stdint.h>

namespace blend {

// Plan sections inside the device plan buffer (blend_plan.off / .count index).
enum PlanSection {
  SEC_TOK_POS = 0,     // int32[T]   absolute position of query token (row of q)
  SEC_ITEM_TOK_OFF,    // int32[n_items+1]
  SEC_ITEM_TOKENS,     // int32[]    global token (row) ids of each item, item-row order
  SEC_ENTRIES,         // KvEntry[E]
  SEC_DENSE_UNITS,     // Unit[n_dense]
  SEC_STREAM_UNITS,    // Unit[n_stream]
  SEC_PARTMAP,         // int32[]    per (item, split) x item token: partial row | DIRECT | SKIP
  SEC_MERGE_TOK,       // int32[M]   tokens with >= 2 sources
  SEC_MERGE_OFF,       // int32[M+1] list m = partial rows merge_off[m] .. merge_off[m+1]-1, ascending
                       //            key-range start (reading #17)
  SEC_STREAM_ROWS,     // RowDesc[n_stream * STREAM_ROWS]  per-row descriptors of the streaming units
  SEC_DENSE_QTOK,      // int32[n_dense]  first token of a dense unit whose tokens are consecutive
                       //                 (its Q tiles load by TMA boxes), else -1
  SEC_DENSE_KS,        // Unit[n_ks]      dense units of <= 128 rows and >= 2 blocks, run key-split
                       //                 by dense_ks.cu (same layout as SEC_DENSE_UNITS)
  SEC_DENSE_KS_QTOK,   // int32[n_ks]     SEC_DENSE_QTOK of those units
  SEC_COUNT
};

constexpr int32_t PM_DIRECT = -1;   // the only source of this token: write out/lse directly
constexpr int32_t PM_SKIP = -2;     // this (item, split) has no key at or before the token

// One KV page entry: <= 64 consecutive slots of one physical page.
struct KvEntry {
  int32_t page;      // physical page id
  int32_t row_off;   // first slot inside the page (0, or 64 when ps = 128)
  int32_t pos0;      // absolute position of slot row_off
  int32_t count;     // valid slots (1..min(ps,64)); slots >= count are masked
};

// One kernel work unit: rows [row_begin, row_begin + n_rows) of an item for one
// kv head, over entries [entry_begin, entry_end).  Item row r = token_local * g + j,
// q head = kvh * g + j.
struct Unit {
  int32_t item;
  int32_t kvh;
  int32_t row_begin;
  int32_t n_rows;
  int32_t entry_begin;
  int32_t entry_end;
  int32_t pm_base;     // partmap index of token_local 0 for this (item, split)
  int32_t tok_base;    // item_tok_off[item]
};

// Row r of a streaming unit, precomputed by the planner (padding rows: qrow = -1).
struct RowDesc {
  int32_t qrow;      // token * Hq + q head: row of q / out / lse
  int32_t pos;       // absolute position of the token (causal bound)
  int32_t target;    // partmap value: partial row | PM_DIRECT | PM_SKIP
  int32_t head;      // q head (partial-row column)
};

constexpr int DENSE_ROWS = 256;    // rows per dense unit: two 128-row tcgen05 Q tiles (UMMA M=128)
constexpr int STREAM_ROWS = 16;    // rows per streaming (mma.sync m16) unit
constexpr int ENTRY_MAX = 64;      // slots per KV entry (TMA box rows)

}  // namespace blend
