// assign.cpp -- row f3: greedy device assignment of a strategy.
//
// A configuration only says how a vertex's iteration space is split; which device runs which
// part is left to "a simple greedy assignment that maximizes data locality (i.e. a greedy
// assignment that maximizes |A(v,d,phi) ∩ A(u,d,phi)|)".  DESIGN reading U:
//   * shard s of v = the digits of s in the radix of v's split tuple (dim 0 most significant);
//   * vertices in node-id order, shards in index order; a shard takes the free device that
//     maximises the summed overlap, over edges to already-placed neighbours, between what the
//     consumer shard on that device needs of the producer's output tensor and what the producer
//     shard on that device holds (elements); ties -> lowest device id;
//   * realized t_x of an edge = 2 elem max_d (|needed on d| - |needed on d ∩ held
//     on d|) bytes over the devices d holding a consumer shard.
// The aligned t_x of the cost model (reading K) is a lower bound of the realized one (per axis
// an overlap never exceeds min(need, held)); it is reached on chains, not always on branchy
// graphs (tests/test_assign.py).  Host-side integer work, O(|V| p^2 deg axes): a post-process
// of the strategy, not part of the search.
#include <algorithm>
#include <cstdint>
#include <string>
#include <vector>

#include "pase_internal.h"

namespace pase {

namespace {
struct Interval { int64_t lo, hi; };

int64_t meet(const Interval& a, const Interval& b) {
    const int64_t lo = std::max(a.lo, b.lo), hi = std::min(a.hi, b.hi);
    return hi > lo ? hi - lo : 0;
}
}  // namespace

pase_status assign_devices(const Plan& P, const int32_t* config_index, int32_t* device_out, double* tx_out,
                           std::string& err) {
    const int n = P.n, m = P.m, p = P.p;
    // chosen tuples and shard digits
    std::vector<const int32_t*> tup(n);
    std::vector<int> nshard(n);
    std::vector<std::vector<int32_t>> digit(n);          // [s * dims + k]
    for (int v = 0; v < n; ++v) {
        const int c = config_index[v];
        if (c < 0 || c >= P.K[v]) {
            err = "pase_assign_devices: node " + std::to_string(v) + ": config index " + std::to_string(c) +
                  " outside [0, " + std::to_string(P.K[v]) + ")";
            return PASE_ERR_INVALID;
        }
        tup[v] = &P.cfg[(size_t)(P.cfg_off[v] + c) * kMaxDims];
        const int dims = P.nodes[v].n_dims;
        int s = 1;
        for (int k = 0; k < dims; ++k) s *= tup[v][k];
        if (s > p) { err = "pase_assign_devices: internal: more shards than devices"; return PASE_ERR_STATE; }
        nshard[v] = s;
        digit[v].resize((size_t)s * dims);
        for (int x = 0; x < s; ++x) {
            int r = x;
            for (int k = dims - 1; k >= 0; --k) { digit[v][(size_t)x * dims + k] = r % tup[v][k]; r /= tup[v][k]; }
        }
    }
    // per edge and output axis: the producer's held interval per producer shard and the
    // consumer's needed interval per consumer shard
    struct EdgeIv { std::vector<Interval> held, need; int axes; };   // [shard * axes + a]
    std::vector<EdgeIv> iv(m);
    std::vector<std::vector<int>> inc(n);
    for (int e = 0; e < m; ++e) {
        const pase_edge& ed = P.edges[e];
        const pase_node& u = P.nodes[ed.src];
        const int A = u.n_out_axes;
        const int du = u.n_dims, dw = P.nodes[ed.dst].n_dims;
        EdgeIv& x = iv[e];
        x.axes = A;
        x.held.resize((size_t)nshard[ed.src] * A);
        x.need.resize((size_t)nshard[ed.dst] * A);
        for (int s = 0; s < nshard[ed.src]; ++s)
            for (int a = 0; a < A; ++a) {
                const int k = u.out_axes[a];
                const int64_t h = u.size[k] / tup[ed.src][k];
                const int64_t lo = digit[ed.src][(size_t)s * du + k] * h;
                x.held[(size_t)s * A + a] = {lo, lo + h};
            }
        for (int s = 0; s < nshard[ed.dst]; ++s)
            for (int a = 0; a < A; ++a) {
                const int64_t ext = u.size[u.out_axes[a]];
                const int mp = ed.axis_map[a];
                if (mp < 0) { x.need[(size_t)s * A + a] = {0, ext}; continue; }
                const int64_t cnt = tup[ed.dst][mp];
                const int64_t part = (ext + cnt - 1) / cnt;
                const int64_t lo = std::min(ext, digit[ed.dst][(size_t)s * dw + mp] * part);
                x.need[(size_t)s * A + a] = {lo, std::min(ext, lo + part)};   // empty past the end
            }
        inc[ed.src].push_back(e);
        inc[ed.dst].push_back(e);
    }
    auto overlap = [&](int e, int su, int sw) -> int64_t {       // held(su) ∩ need(sw)
        const EdgeIv& x = iv[e];
        int64_t o = 1;
        for (int a = 0; a < x.axes && o; ++a) o *= meet(x.held[(size_t)su * x.axes + a], x.need[(size_t)sw * x.axes + a]);
        return o;
    };
    auto need_vol = [&](int e, int sw) -> int64_t {
        const EdgeIv& x = iv[e];
        int64_t o = 1;
        for (int a = 0; a < x.axes; ++a) o *= x.need[(size_t)sw * x.axes + a].hi - x.need[(size_t)sw * x.axes + a].lo;
        return o;
    };
    // greedy placement
    std::vector<int32_t> on(n * (size_t)p, -1);                 // shard of v on device d
    std::vector<char> placed(n, 0);
    std::vector<int64_t> score(p);
    for (int v = 0; v < n; ++v) {
        for (int s = 0; s < nshard[v]; ++s) {
            std::fill(score.begin(), score.end(), 0);
            for (int e : inc[v]) {
                const pase_edge& ed = P.edges[e];
                const int other = ed.src == v ? ed.dst : ed.src;
                if (!placed[other]) continue;
                for (int d = 0; d < p; ++d) {
                    const int t = on[(size_t)other * p + d];
                    if (t < 0) continue;
                    score[d] += ed.src == v ? overlap(e, s, t) : overlap(e, t, s);
                }
            }
            int best = -1;
            for (int d = 0; d < p; ++d)
                if (on[(size_t)v * p + d] < 0 && (best < 0 || score[d] > score[best])) best = d;
            on[(size_t)v * p + best] = s;
            if (device_out) device_out[(size_t)v * p + s] = best;
        }
        if (device_out)
            for (int s = nshard[v]; s < p; ++s) device_out[(size_t)v * p + s] = -1;
        placed[v] = 1;
    }
    if (tx_out)
        for (int e = 0; e < m; ++e) {
            const pase_edge& ed = P.edges[e];
            int64_t worst = 0;
            for (int d = 0; d < p; ++d) {
                const int sw = on[(size_t)ed.dst * p + d];
                if (sw < 0) continue;
                const int su = on[(size_t)ed.src * p + d];
                worst = std::max(worst, need_vol(e, sw) - (su >= 0 ? overlap(e, su, sw) : 0));
            }
            tx_out[e] = (double)(uint64_t)(2 * (int64_t)P.nodes[ed.src].elem_bytes * worst);
        }
    return PASE_OK;
}

}  // namespace pase
