// Byte-exact device / host footprint formulas of the B200 engine. Shared by
// the device arena (which allocates exactly this) and the planner-style
// reports, so "plan == ledger" holds by construction (reference
// proj/include/hlm/footprint.hpp:22-87 plays the same role).
//
// Differences from the reference layout, all consequences of the GPU design:
//   * activations: bf16 GEMM operands + fp32 residual, flash attention keeps
//     O and the row log-sum-exp instead of the (B,S,S) probability matrix;
//   * outbound gradients are fp32 and double-buffered so the D2H copy of
//     layer i overlaps the backward of layer i-1.
#pragma once

#include <cstddef>

#include "hlm/model_config.hpp"
#include "hlm_cuda.h"

namespace hlm {
inline namespace b200 {

inline HlmBlockDims block_dims(const ModelConfig& m, int flags = 0) {
    HlmBlockDims d{};
    d.batch = m.batch;
    d.seq = m.seq;
    d.hidden = m.hidden;
    d.ffn = m.ffn;
    d.n_heads = static_cast<int32_t>(m.n_heads);
    d.flags = flags;
    return d;
}

// One block's saved activations (A_max): n1, q|k|v, o, lse, y, n2, up|gate, act.
inline i64 block_act_bytes(const ModelConfig& m) {
    const HlmBlockDims d = block_dims(m);
    return static_cast<i64>(hlm_cuda_block_acts_bytes(&d));
}

// One checkpoint anchor: the fp32 (batch, seq, hidden) residual stream.
inline i64 anchor_slot_bytes(const ModelConfig& m) { return 4 * m.rows() * m.hidden; }

// One weight stream buffer: the widest tile in bf16 (rounded to 256 B).
inline i64 stream_buf_bytes(const ModelConfig& m) { return (2 * m.max_tile_params() + 255) / 256 * 256; }

// One outbound fp32 gradient buffer (device) / one host slab: the widest tile.
inline i64 grad_buf_bytes(const ModelConfig& m) { return (4 * m.max_tile_params() + 255) / 256 * 256; }

inline i64 align256(i64 x) { return (x + 255) / 256 * 256; }

struct WorkspaceLayout {
    i64 g_roll = 0;       // 2 x (rows, h) fp32 gradient carry
    i64 h_roll = 0;       // 2 x (rows, h) fp32 rolling state (K > 1 recompute)
    i64 block_ws = 0;     // block backward scratch
    i64 head_ws = 0;      // bf16 x, fp32 logits, bf16 d_logits
    i64 grad_out = 0;     // 2 x widest tile fp32
    i64 discard_acts = 0; // forward-pass activations (not kept)
    i64 misc = 0;         // tokens, targets, CSR, loss rows, RoPE tables, flags
    i64 total() const { return g_roll + h_roll + block_ws + head_ws + grad_out + discard_acts + misc; }
};

inline WorkspaceLayout workspace_layout(const ModelConfig& m) {
    WorkspaceLayout w;
    const i64 T = m.rows(), h = m.hidden;
    const HlmBlockDims d = block_dims(m);
    w.g_roll = 2 * align256(4 * T * h);
    w.h_roll = 2 * align256(4 * T * h);
    w.block_ws = align256(static_cast<i64>(hlm_cuda_block_ws_bytes(&d)));
    w.head_ws = align256(static_cast<i64>(hlm_cuda_head_ws_bytes(T, h, m.vocab)));
    w.grad_out = 2 * grad_buf_bytes(m);
    w.discard_acts = align256(block_act_bytes(m));
    const i64 hd = m.head_dim();
    w.misc = 2 * align256(4 * T) + align256(4 * (m.vocab + 1)) + align256(4 * T) + align256(4 * T) +
             2 * align256(4 * m.seq * (hd / 2 > 0 ? hd / 2 : 1)) + 256;
    return w;
}

struct ArenaFootprint {
    i64 stream_buf = 0;    // per buffer
    i64 stream_buf_block = 0;   // one block tile in bf16 (a weight-cache slot)
    i64 weight_cache = 0;  // optional HBM weight cache (multiple of stream_buf_block)
    i64 anchor_slot = 0;   // per anchor
    i64 anchor_slots = 0;  // ceil(L/K) + 1
    i64 stack = 0;         // K x (A_max + fp32 block output)
    i64 workspace = 0;
    i64 anchors_total() const { return anchor_slots * anchor_slot; }
    i64 core_total() const { return 2 * stream_buf + stack + workspace + weight_cache; }
    i64 total() const { return core_total() + anchors_total(); }
};

inline ArenaFootprint arena_footprint(const ModelConfig& m, i64 weight_cache_bytes = 0) {
    ArenaFootprint fp;
    fp.stream_buf = stream_buf_bytes(m);
    fp.stream_buf_block = (2 * m.block_params() + 255) / 256 * 256;
    i64 slots = weight_cache_bytes / fp.stream_buf_block;
    if (slots > m.layers) slots = m.layers;
    fp.weight_cache = slots * fp.stream_buf_block;
    fp.anchor_slot = align256(anchor_slot_bytes(m));
    fp.anchor_slots = m.anchor_capacity();
    // each stack slab: the block's activations + its fp32 output (the next
    // layer's input while a K-group is recomputed)
    fp.stack = m.k_ckpt * (align256(block_act_bytes(m)) + align256(anchor_slot_bytes(m)));
    fp.workspace = workspace_layout(m).total();
    return fp;
}

// Persistent host bytes per parameter: fp32 master + m + v, bf16 shadow.
inline i64 persistent_bytes_per_param() { return 14; }

}  // inline namespace b200
}  // namespace hlm
