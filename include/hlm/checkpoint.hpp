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
// Loads into a store of identical geometry; throws ConfigError otherwise.
void load_checkpoint(MasterStore& store, const std::string& path);

}  // inline namespace b200
}  // namespace hlm
