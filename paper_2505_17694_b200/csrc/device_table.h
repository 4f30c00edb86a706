// Layout of the int32 task-table blob shared by host_table.cpp (writer)
// and the kernels (readers). See codec_table_build in codec_b200.h.
#pragma once

#include <cstdint>

namespace codec {

// group kinds (which kernel runs the group)
constexpr int kKindTc = 0;       // tcgen05 shared-node kernel (bf16, d = 128)
constexpr int kKindGemv = 1;     // CUDA-core warp-shuffle GEMV kernel
constexpr int kKindGeneric = 2;  // any dtype / head dim (small or odd shapes)
constexpr int kKindMulti = 3;    // multi-request mma.sync kernel: 2..kMultiRows/g requests of one slice
constexpr int kKindTct = 4;      // transposed tcgen05 kernel (kern_tct.cu): up to kTctRows rows of one slice

// a group record: 8 int32
constexpr int kGroupInts = 8;
constexpr int kGrpKvTok = 0;    // pool token index of the slice start
constexpr int kGrpLen = 1;      // slice length (tokens)
constexpr int kGrpRowBegin = 2; // first row record
constexpr int kGrpNRows = 3;    // number of requests in the group
constexpr int kGrpMaxVis = 4;   // most visible tokens of any row (kernels size their tile loop by it)
constexpr int kGrpNode = 5;     // GEMV / generic: forest node (diagnostics)
constexpr int kGrpQReq0 = 5;    // TC pieces: first request of a consecutive request run (Q by TMA), else -1
constexpr int kGrpBlock = 6;    // TC: schedule block (CTA pair) of the unit
constexpr int kGrpStart = 6;    // GEMV / generic: slice start within the node (host-side growth)
constexpr int kGrpHead = 7;     // TC: local kv head of the unit

// a row record: 4 int32 -- request, visible tokens within the slice,
// partial slot (>= 0) or -1 - request for a direct write of the output
constexpr int kRowInts = 4;

// minimum query-head rows for a subtask to take the tensor-core kernel
// (without the multi-request kernel: CODEC_FLAG_NO_MULTI, or shapes it
// does not cover)
constexpr int kTcMinRows = 16;
// with the multi-request kernel: slices of up to kMultiMaxRows query-head
// rows take it (in groups of kMultiRows rows), larger ones the tensor cores
constexpr int kMultiRows = 32;
#ifndef CODEC_MULTI_MAX_ROWS
#define CODEC_MULTI_MAX_ROWS 16
#endif
constexpr int kMultiMaxRows = CODEC_MULTI_MAX_ROWS;
// transposed tensor-core kernel: slices of 2+ requests of nodes with at
// most kTctMaxRows query-head rows (CODEC_TCT_MAX_ROWS overrides;
// CODEC_FLAG_TCT_WIDE raises it to kTctRows), in groups of at most kTctRows
// rows (the MMA's N; groups of up to 64 rows run the narrow variant, 65..128
// the wide one); larger nodes take the M = 256 pair kernel
constexpr int kTctRows = 128;
#ifndef CODEC_TCT_MAX_ROWS
#define CODEC_TCT_MAX_ROWS 64
#endif
constexpr int kTctMaxRows = CODEC_TCT_MAX_ROWS;
// query-head rows of one tensor-core group (M = 256: one 128-row tile per
// CTA of a cta_group::2 pair)
constexpr int kTcGroupRows = 256;
// SMs (CTAs) that run one tensor-core schedule block
constexpr int kTcCtasPerBlock = 2;
// device balancer: a unit boundary inside a CTA pair costs this many KV
// tiles (host_table.cpp; CODEC_TC_UNIT_COST overrides)
constexpr int kTcUnitCostDefault = 0;

// debug CTA log (CODEC_FLAG_CTALOG): TC records first, GEMV from this index
constexpr int kCtaLogGemv = 4096;
constexpr int kCtaLogLen = 4096 + 65536;

}  // namespace codec
