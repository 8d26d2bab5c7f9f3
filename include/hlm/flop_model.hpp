// Flop accounting. The reference model (proj/include/hlm/flop_model.hpp:14-32:
// fwd = 2 n T, bwd = 2 fwd, recompute = fwd, no attention) is kept for
// trace compatibility; MODEL_FLOPS / HW_FLOPS follow SURVEY.md §8(d) and add
// causal-attention matmul flops.
#pragma once

#include "hlm/model_config.hpp"

namespace hlm {
inline namespace b200 {

inline i64 fwd_flops(i64 n_params, i64 tokens) { return 2 * n_params * tokens; }
inline i64 bwd_flops(i64 n_params, i64 tokens) { return 2 * fwd_flops(n_params, tokens); }

// Causal attention matmul flops of one block forward: QK^T and PV over the
// lower triangle: 2 * B * S^2 * h.
inline double attn_fwd_flops(const ModelConfig& m) {
    return 2.0 * static_cast<double>(m.batch) * static_cast<double>(m.seq) * static_cast<double>(m.seq) *
           static_cast<double>(m.hidden);
}

// MODEL_FLOPS = 6 T (L n_mm + V h) + 6 L B S^2 h
inline double model_flops(const ModelConfig& m) {
    const double T = static_cast<double>(m.rows());
    return 6.0 * T * (static_cast<double>(m.layers) * static_cast<double>(m.block_matmul_params()) +
                      static_cast<double>(m.vocab) * static_cast<double>(m.hidden)) +
           3.0 * static_cast<double>(m.layers) * attn_fwd_flops(m);
}

// HW_FLOPS = MODEL_FLOPS + L (2 n_mm T + 2 B S^2 h)  (per-layer recompute)
inline double hw_flops(const ModelConfig& m) {
    const double T = static_cast<double>(m.rows());
    return model_flops(m) + static_cast<double>(m.layers) *
                                (2.0 * static_cast<double>(m.block_matmul_params()) * T + attn_fwd_flops(m));
}

}  // inline namespace b200
}  // namespace hlm
