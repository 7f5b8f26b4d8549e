// Host-side frontier expansion (see mcsg_frontier.cpp).
#pragma once
#include <cstdint>
#include <vector>

#include "mcsg_device.h"

namespace mcsg {

struct Frontier {
    std::vector<TaskSlot> tasks;  // disjoint subtrees covering the whole search tree (n <= 64)
    std::vector<WideSlot> wtasks; // the same for wide instances
    uint64_t nodes = 0;           // nodes entered on the host
    int best_size = 0;            // host incumbent (mapping below)
    std::vector<uint8_t> best_v, best_u;
    bool max_reached = false;     // the host already found a mapping of size min(n_G, n_H)
};

// Breadth-first expansion until at least `target` open subtrees exist (or the
// tree is exhausted). `d` must be packed in the kernel's vertex order.
Frontier expand_frontier(const InstanceDesc& d, bool directed, int target, int inst);
Frontier expand_frontier(const WideDesc& d, bool directed, int target, int inst);

}  // namespace mcsg
