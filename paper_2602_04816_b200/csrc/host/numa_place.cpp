// NUMA-aware CPU partition and page placement for data-parallel ranks
// (see include/hlm/numa_place.hpp).
#include "hlm/numa_place.hpp"

#include <cuda_runtime.h>
#include <sched.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <cctype>
#include <cstdint>
#include <fstream>
#include <sstream>
#include <string>

namespace hlm {
inline namespace b200 {
namespace {

constexpr int kMpolPreferred = 1;   // linux/mempolicy.h

std::string read_line(const std::string& path) {
    std::ifstream f(path);
    std::string s;
    if (f) std::getline(f, s);
    return s;
}

// "0-3,8,10-11" -> {0,1,2,3,8,10,11}
std::vector<int> parse_cpulist(const std::string& s) {
    std::vector<int> out;
    std::stringstream ss(s);
    std::string part;
    while (std::getline(ss, part, ',')) {
        if (part.empty()) continue;
        const auto dash = part.find('-');
        try {
            if (dash == std::string::npos) {
                out.push_back(std::stoi(part));
            } else {
                const int a = std::stoi(part.substr(0, dash)), b = std::stoi(part.substr(dash + 1));
                for (int c = a; c <= b; ++c) out.push_back(c);
            }
        } catch (...) {
            return {};
        }
    }
    std::sort(out.begin(), out.end());
    return out;
}

}  // namespace

int numa_node_count() {
    int n = 0;
    while (!read_line("/sys/devices/system/node/node" + std::to_string(n) + "/cpulist").empty()) ++n;
    return std::max(n, 1);
}

int gpu_numa_node(int device) {
    char bus[32] = {};
    if (cudaDeviceGetPCIBusId(bus, sizeof bus, device) != cudaSuccess) {
        (void)cudaGetLastError();
        return -1;
    }
    std::string id(bus);
    for (auto& ch : id) ch = static_cast<char>(std::tolower(static_cast<unsigned char>(ch)));
    const std::string s = read_line("/sys/bus/pci/devices/" + id + "/numa_node");
    if (s.empty()) return -1;
    try {
        return std::stoi(s);   // -1 on single-node hosts
    } catch (...) {
        return -1;
    }
}

std::vector<int> node_cpus(int node) {
    if (node < 0) return {};
    return parse_cpulist(read_line("/sys/devices/system/node/node" + std::to_string(node) + "/cpulist"));
}

std::vector<int> allowed_cpus() {
    cpu_set_t set;
    CPU_ZERO(&set);
    std::vector<int> out;
    if (sched_getaffinity(0, sizeof(set), &set) != 0) return out;
    for (int c = 0; c < CPU_SETSIZE; ++c)
        if (CPU_ISSET(c, &set)) out.push_back(c);
    return out;
}

std::vector<int> rank_cpu_slice(int rank, const std::vector<int>& nodes, const std::vector<int>& allowed,
                                int online, const std::vector<std::vector<int>>& cpus_of_node) {
    const int world = static_cast<int>(nodes.size());
    if (world <= 1 || allowed.empty() || static_cast<int>(allowed.size()) < online) return allowed;
    const int my = nodes[static_cast<size_t>(rank)];
    std::vector<int> pool;
    std::vector<int> group;
    if (my >= 0 && static_cast<size_t>(my) < cpus_of_node.size()) {
        for (int c : cpus_of_node[static_cast<size_t>(my)])
            if (std::binary_search(allowed.begin(), allowed.end(), c)) pool.push_back(c);
        for (int r = 0; r < world; ++r)
            if (nodes[static_cast<size_t>(r)] == my) group.push_back(r);
    }
    if (pool.empty()) {   // node unknown: split the whole set among all ranks
        pool = allowed;
        group.clear();
        for (int r = 0; r < world; ++r) group.push_back(r);
    }
    const size_t g = group.size(), idx = static_cast<size_t>(std::find(group.begin(), group.end(), rank) - group.begin());
    const size_t C = pool.size(), lo = idx * C / g, hi = (idx + 1) * C / g;
    if (hi <= lo) return {pool[idx % C]};
    return std::vector<int>(pool.begin() + static_cast<long>(lo), pool.begin() + static_cast<long>(hi));
}

std::vector<int> rank_gpu_nodes(int world) {
    std::vector<int> nodes(static_cast<size_t>(std::max(world, 0)), -1);
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess) {
        (void)cudaGetLastError();
        return nodes;
    }
    if (ndev < world) return nodes;
    for (int r = 0; r < world; ++r) nodes[static_cast<size_t>(r)] = gpu_numa_node(r % ndev);
    return nodes;
}

bool prefer_node(void* addr, std::size_t bytes, int node) {
    if (node < 0 || node >= 64 || numa_node_count() < 2) return true;
    const std::uintptr_t page = static_cast<std::uintptr_t>(sysconf(_SC_PAGESIZE));
    const std::uintptr_t a = reinterpret_cast<std::uintptr_t>(addr);
    const std::uintptr_t lo = (a + page - 1) / page * page, hi = (a + bytes) / page * page;
    if (hi <= lo) return true;
    unsigned long mask = 1UL << node;
    return syscall(SYS_mbind, lo, hi - lo, kMpolPreferred, &mask, sizeof(mask) * 8, 0) == 0;
}

ScopedPreferNode::ScopedPreferNode(int node) {
    if (node < 0 || node >= 64 || numa_node_count() < 2) return;
    unsigned long mask = 1UL << node;
    active_ = syscall(SYS_set_mempolicy, kMpolPreferred, &mask, sizeof(mask) * 8) == 0;
}

ScopedPreferNode::~ScopedPreferNode() {
    if (active_) (void)syscall(SYS_set_mempolicy, 0 /* MPOL_DEFAULT */, nullptr, 0);
}

}  // inline namespace b200
}  // namespace hlm
