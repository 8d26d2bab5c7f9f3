// Host placement for data-parallel ranks sharing one host store.
//
// Each rank runs the host Adam of its 1/world shard of every tile with an
// OpenMP team; N ranks on one host must not pin N full-size teams onto the same
// CPUs, and on a multi-socket host a rank's shard (master, m, v, shadow) should
// live in the DRAM of the socket its GPU and its team sit on. Ranks map to
// devices as rank % device_count (the LOCAL_RANK convention of the launcher).
// Everything here is best effort: with one NUMA node, no sysfs, or a launcher
// that already bound the process, it degrades to a plain partition / no-op.
#pragma once

#include <cstddef>
#include <vector>

namespace hlm {
inline namespace b200 {

int numa_node_count();                        // nodes under /sys/devices/system/node (>= 1)
int gpu_numa_node(int device);                // -1 when unknown
std::vector<int> node_cpus(int node);         // sorted CPU ids of a node; empty when unknown
std::vector<int> allowed_cpus();              // this process's affinity set, sorted

// CPUs this rank's optimizer team may use: the rank's share of the CPUs of its
// GPU's NUMA node, split evenly among the ranks whose GPUs sit on the same node.
// `allowed` is the process affinity, `online` the host's CPU count, `nodes[r]`
// the NUMA node of rank r's GPU (-1 unknown). A process already bound to fewer
// CPUs than the host has keeps its whole set (the launcher placed it).
std::vector<int> rank_cpu_slice(int rank, const std::vector<int>& nodes, const std::vector<int>& allowed,
                                int online, const std::vector<std::vector<int>>& cpus_of_node);

// NUMA node of each rank's GPU (rank % device_count); all -1 when fewer devices
// than ranks are visible (one GPU per process: the mapping is unknown).
std::vector<int> rank_gpu_nodes(int world);

// Prefer `node` for the pages of [addr, addr + bytes) not yet touched (whole
// pages inside the range). No-op for node < 0 or a single-node host. Returns
// false when the kernel refused the policy.
bool prefer_node(void* addr, std::size_t bytes, int node);

// While alive, new pages faulted by this thread prefer `node` (the rank's pinned
// gradient slabs are allocated under it). No-op for node < 0 or one node.
class ScopedPreferNode {
public:
    explicit ScopedPreferNode(int node);
    ~ScopedPreferNode();
    ScopedPreferNode(const ScopedPreferNode&) = delete;
    ScopedPreferNode& operator=(const ScopedPreferNode&) = delete;

private:
    bool active_ = false;
};

}  // inline namespace b200
}  // namespace hlm
