// Host-side graph core for the drop-in (see mcsg_graph.cpp for citations).
#pragma once
#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/mcsg.h"
#include "mcsg_device.h"

namespace mcsg {

// GraphError (graph.hpp:25-28) / ParseError (graph_io.hpp:11) counterparts.
struct Error : std::runtime_error {
    explicit Error(const std::string& w) : std::runtime_error(w) {}
};
struct ParseErr : Error {
    explicit ParseErr(const std::string& w) : Error(w) {}
};

struct HostGraph {
    int n = 0;
    bool directed = false;
    bool labeled = false;
    std::vector<uint8_t> codes;   // n*n row-major (graph.hpp:60)
    std::vector<int32_t> labels;

    uint8_t code(int u, int v) const { return codes[size_t(u) * n + v]; }
    int degree(int v) const;
    HostGraph permuted(const std::vector<int>& fwd) const;  // permute(), graph.cpp:94-109
    static HostGraph from_abi(const mcsg_graph* g);
};

void random_graph(int n, double density, uint64_t seed, bool directed, int label_count,
                  uint8_t* codes, int32_t* labels);
std::vector<int> random_permutation(int n, uint64_t seed);
std::vector<int> make_ordering(const HostGraph& g, int strategy);
int verify(const HostGraph& g, const HostGraph& h, const int32_t* pairs, int k);

HostGraph load_mivia(const std::vector<uint8_t>& bytes);
std::vector<uint8_t> save_mivia(const HostGraph& g);
HostGraph load_text(const std::string& text);
std::string save_text(const HostGraph& g);
HostGraph load_graph_file(const std::string& path, int format);
void save_graph_file(const HostGraph& g, const std::string& path, int format);

void pack_instance(const HostGraph& g, const HostGraph& h, int goal, bool prune, int floor_size,
                   int group, InstanceDesc* d);
void pack_wide(const HostGraph& g, const HostGraph& h, int goal, bool prune, int floor_size, int group,
               WideDesc* d);

}  // namespace mcsg
