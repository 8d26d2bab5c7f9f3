// HLM2: on-disk image of the B200 host store (the mixed-precision layout:
// FP32 master, FP32 m, FP32 v per physical tile; the BF16 shadow is re-derived
// on load). Successor of reference HLM1 (proj/src/checkpoint.cpp:15-120): same
// little-endian header style, 4096-aligned raw tile payloads, strict geometry
// checks on load, Adam step count carried so a resumed run_training replays
// the data stream (trainer.cpp:18-19) and continues bitwise.
#pragma once

#include <string>

#include "hlm/host_store.hpp"

namespace hlm {
inline namespace b200 {

void save_checkpoint(const MasterStore& store, const std::string& path);
// Loads into a store of identical geometry; throws ConfigError otherwise. Reads HLM2
// and the reference's HLM1 (proj/src/checkpoint.cpp:71-120, same checks and messages):
// master := the HLM1 weights (exact for BF16), m and v restored, the Adam step count
// restored; HLM1's gradient region (last-step scratch) is not used.
void load_checkpoint(MasterStore& store, const std::string& path);
// Writes the reference's HLM1 container (proj/src/checkpoint.cpp:38-69) so the
// reference's load_checkpoint reads it: weights in the store dtype (BF16: the shadow,
// RNE of the master), gradients in the store dtype (zeros when the store holds none),
// FP32 m and v, the Adam step count.
void save_checkpoint_hlm1(const MasterStore& store, const std::string& path);

}  // inline namespace b200
}  // namespace hlm
