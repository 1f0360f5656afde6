// pase_internal.h -- internal types shared by the host core (host.cpp), the C ABI
// (capi.cu) and the sm_100a kernels (kernels.cu).  Not installed; include/pase.h is
// the public boundary.  Citations: P:<n> = PAPER.md line n.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "pase.h"

namespace pase {

constexpr int kMaxDims = PASE_MAX_DIMS;
constexpr int kMaxDep = PASE_MAX_DEP;

// ---------------------------------------------------------------------------------
// Host plan (a1-a4): everything pase_create derives from the graph, before the GPU.
// ---------------------------------------------------------------------------------
struct Plan {
    int n = 0, m = 0, p = 1, policy = 0;
    double r = 0.0;                              // F / B
    std::vector<pase_node> nodes;
    std::vector<pase_edge> edges;

    // a2: C(v) -- per node K_v and its tuples (row-major, kMaxDims int32 per config)
    std::vector<int32_t> K;
    std::vector<int64_t> cfg_off;                // n+1, in configs
    std::vector<int32_t> cfg;                    // cfg_off[n] * kMaxDims

    // a3: SortNodes (Fig. 4): sigma (rank -> node), rank (node -> rank), D(i) by rank
    std::vector<int32_t> sigma, rank;
    std::vector<std::vector<int32_t>> dep;       // D(i) node ids, ascending rank

    // a4: elimination tree over ranks, E>(sigma_i), levels
    std::vector<int32_t> parent;                 // rank of min-rank D(i), -1 for root
    std::vector<std::vector<int32_t>> children;  // ranks, ascending
    std::vector<std::vector<int32_t>> egt;       // edge ids, by (rank(other end), edge id)
    std::vector<int32_t> level;                  // 0 = leaves
    int levels = 0;

    // layout: per rank |T(i)|, offsets into the T / A pools (entries)
    std::vector<int64_t> tsize, toff;
    std::vector<int64_t> loff;                   // n+1: L_v offset (doubles)
    std::vector<int64_t> woff;                   // m+1: W_e offset (doubles)
    int max_dep = 0, max_k = 0;
    uint64_t candidates = 0, entries = 0;
};

// Builds a Plan.  Returns PASE_OK or an error with a message.
pase_status build_plan(const pase_graph* g, int32_t p, const pase_machine* m, Plan& plan,
                       std::string& err);

// ---------------------------------------------------------------------------------
// Device descriptors (kernels.cu)
// ---------------------------------------------------------------------------------
struct EdgeDesc {            // cost-table kernel: one per edge
    int32_t src, dst;
    int32_t later_is_src;    // W row = config of the later-ranked endpoint
    int32_t pad;
    int32_t axis_map[kMaxDims];
    int64_t woff;            // doubles
};

struct TermDesc {            // one summand of Eq. 4 for a vertex (L, one W_e, or one child T_j)
    const double* base;      // element(phi, C) = base[sum_q c_q * stride[q] + C]
    int64_t stride[kMaxDep];
};

struct VertexDesc {          // one DP vertex (rank i)
    int32_t K;               // |C(sigma_i)|, the reduction extent
    int32_t m;               // |D(i)|
    int32_t nterms;          // 1 + |E>(sigma_i)| + |children(i)|, canonical order
    int32_t term0;           // first TermDesc
    int64_t nout;            // |T(i)|
    int32_t radix[kMaxDep];  // K of each D(i) coordinate, ascending rank (lowest fastest)
    double* T;               // output table
    uint16_t* A;             // argmin table
};

// kernels.cu entry points (host-side launchers)
void launch_cost_tables(const pase_node* nodes_dev, const int32_t* K_dev, const int64_t* cfg_off_dev,
                        const int32_t* cfg_dev, const int64_t* loff_dev, int n,
                        const EdgeDesc* edges_dev, int m, const int64_t* item_off_dev,
                        int64_t total, double r, double* L_dev, double* W_dev, void* stream);
void launch_dp_vertex(const VertexDesc* vd_dev, const TermDesc* td_dev, int vertex,
                      const VertexDesc& vd_host, void* stream);
void launch_backtrack(const int32_t* sigma_dev, const int32_t* dep_off_dev, const int32_t* dep_ids_dev,
                      const VertexDesc* vd_dev, int n, int32_t* choice_dev, double* total_dev,
                      void* stream);

}  // namespace pase
