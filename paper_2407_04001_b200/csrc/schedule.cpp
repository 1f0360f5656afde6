// schedule.cpp -- host-side task plan of the persistent DP kernel.
//
// Single GPU: each DP vertex's items are cut into tasks; the task DAG (a task of vertex p
// waits for all tasks of p's children) is list-scheduled on the CTAs of the grid with
// critical-path priority, giving a static claim order that is topological.
//
// Multi-GPU (world G > 1): a table with |T(i)| * 8 >= redundant_below bytes
// and >= 2 coordinates is partitioned by contiguous ranges of its highest-rank coordinate
// u_top(i) (configs [q*K/G, (q+1)*K/G) of u_top on rank q); smaller tables are computed
// redundantly on every rank.  A partitioned child j whose parent p is partitioned on a
// coordinate that is also in D(j) is partitioned identically (u_top(j) = u_top(p), since
// D(j) ⊆ D(p) ∪ {sigma_p}), so p reads only local rows: no communication.  Otherwise the
// child is "broadcast": its tasks write their outputs into every rank's copy of T(j)
// (peer stores over NVLink, fused into the DP kernel) and decrement every rank's pending
// counter of p.  Argmin tables of partitioned vertices are always broadcast, so every rank
// can back-substitute locally.  One global list schedule over all ranks' tasks gives every
// rank a claim order consistent with a single topological order: deadlock-free across
// ranks (the globally earliest unfinished task always has its dependencies done and is
// held or next to be claimed by its rank).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <queue>

#include "pase_internal.h"

namespace pase {

static const bool kWaveTail = !(std::getenv("PASE_WAVE_TAIL") && std::getenv("PASE_WAVE_TAIL")[0] == '0');
// the wave tail's widened lane groups keep at least this many values of C per lane
static const int kTailMinC = std::getenv("PASE_TAIL_MINC") ? std::max(1, std::atoi(std::getenv("PASE_TAIL_MINC"))) : 8;
static const int kTailSmallKMinC = std::getenv("PASE_TAIL_SMALLK_MINC") ? std::max(1, std::atoi(std::getenv("PASE_TAIL_SMALLK_MINC"))) : kTailMinC;

// Task-duration model of the list schedule: a fixed latency plus candidates at a per-tile-family
// rate (us, candidates per us per CTA).  PASE_DUR="f:a:rate,..." overrides family f (A/B only).
int dur_family(const VertexDesc& d) {
    if (d.shape < 0) return kDurGeneric;
    if (d.wlog > 0) return kDurLatency;
    if (d.shape < kShape2D) return kDur1D;
    if (d.shape < kShape2S) return kDur2D;
    if (d.shape < kShapeG1) return kDur2S;
    if (d.shape < kShapeStream) return kDurG1;
    if (d.shape < kShapeCta) return kDurStream;
    return kDurCta;
}
const DurModel& dur_model() {
    static const DurModel m = [] {
        DurModel r;
        for (int f = 0; f < kDurFamilies; ++f) { r.a[f] = 3.0; r.rate[f] = 3000.0; }
        if (const char* e = std::getenv("PASE_DUR")) {
            int f;
            double a, rate;
            for (const char* q = e; q && *q;) {
                if (std::sscanf(q, "%d:%lf:%lf", &f, &a, &rate) == 3 && f >= 0 && f < kDurFamilies && rate > 0) {
                    r.a[f] = a;
                    r.rate[f] = rate;
                }
                q = std::strchr(q, ',');
                if (q) ++q;
            }
        }
        return r;
    }();
    return m;
}

pase_status build_schedule(const Plan& P, std::vector<VertexDesc>& vd, int world, int rank, int nblocks,
                           SchedPlan& out, std::string& err, const std::vector<int32_t>* chunk_consumer,
                           bool simulate) {
    const int n = P.n;
    const int G = std::max(world, 1);
    nblocks = std::max(nblocks, 1);
    // tasks per CTA of the grid for big vertices: 3 (same-binary A/B against kTasksPerBlock = 4,
    // profiles/r02_ab_reentry.txt: DP -1.3 % Transformer, -2 % LE_P / GNMT 4+4, neutral elsewhere)
    static const int64_t tpb = std::getenv("PASE_TASKS_PER_BLOCK") ? std::atoll(std::getenv("PASE_TASKS_PER_BLOCK")) : 3;
    const int64_t spread = std::max<int64_t>(1, tpb) * nblocks;
    const auto tt0 = std::chrono::steady_clock::now();
    // ---- per (vertex, rank): unit runs, split into tasks
    struct GTask { int32_t rank, vtx; int64_t i0, i1; int32_t glog; };   // glog 0 = the vertex's
    std::vector<GTask> all;
    {
        int64_t est = 0;                                // reserve: ~ items / spread tasks per vertex
        for (int i = 0; i < n; ++i) {
            const int64_t units = vd[i].shape >= 0 ? vd[i].nitems : vd[i].nout;
            const int64_t groups = std::max<int64_t>(1, (256 >> vd[i].glog) >> vd[i].wlog);
            est += std::min<int64_t>(spread, (units + groups - 1) / groups) + 2;
        }
        all.reserve((size_t)(est * G + 16));
    }
    // tasks_of[i] for DP vertex i; tasks_of[n + i] = the cost-table chunks vertex i reads (run by
    // every rank: each needs the full L / W tables), which its tasks wait for like children
    const int nv = chunk_consumer ? 2 * n : n;
    // (vertex, rank) -> its tasks: a counting sort of `all` by vtx * G + rank after it is built
    // (no per-vertex vectors: the host plan is on the end-to-end path)
    std::vector<int32_t> toff((size_t)nv * G + 1, 0), tidx;
    struct Span {
        const int32_t* b;
        const int32_t* e;
        const int32_t* begin() const { return b; }
        const int32_t* end() const { return e; }
        size_t size() const { return (size_t)(e - b); }
        bool empty() const { return b == e; }
        int32_t operator[](size_t k) const { return b[k]; }
    };
    auto tasks_of = [&](int v, int q) { return Span{tidx.data() + toff[(size_t)v * G + q], tidx.data() + toff[(size_t)v * G + q + 1]}; };
    for (int i = 0; i < n; ++i) {
        const VertexDesc& d = vd[i];
        const int64_t units = d.shape >= 0 ? d.nitems : d.nout;
        const int64_t groups = (256 >> d.glog) >> d.wlog;   // items a CTA runs concurrently
        for (int q = 0; q < G; ++q) {
            std::vector<std::pair<int64_t, int64_t>> runs;
            if (!d.part) {
                runs.push_back({0, units});
            } else {
                const int top = d.m - 1;
                const int64_t Kt = d.radix[top];
                const int64_t lo = q * Kt / G, hi = (q + 1) * Kt / G;
                if (d.shape >= 0) {              // items: [low combos] fastest, tile, top (split_item)
                    const int64_t S = d.ncombo / Kt;
                    if (hi > lo) runs.push_back({lo * S * d.ntile, hi * S * d.ntile});
                } else {                         // items = outputs; top is the slowest coordinate
                    const int64_t S = d.nout / Kt;
                    if (hi > lo) runs.push_back({lo * S, hi * S});
                }
            }
            int64_t local = 0;
            for (auto& r : runs) local += r.second - r.first;
            int64_t ti = std::max<int64_t>(groups, (local + spread - 1) / spread);
            ti = (ti + groups - 1) / groups * groups;
            // wave tail: a vertex of one-round tasks spanning more than one wave of
            // the grid leaves a partial last wave whose tasks take as long as full ones.  Those
            // items go to tasks with wider lane groups (the largest G' <= 32 that still fits
            // them in one wave, keeping >= 8 values of C per lane): K/G' serial iterations
            // instead of K/G.  Same items, same results.
            int64_t bulk_end = -1;
            int32_t tail_glog = 0;
            if (kWaveTail && runs.size() == 1 && d.shape >= 0 && d.shape < kShapeG1 && d.wlog == 0 && d.glog < 5 && ti == groups) {
                const int64_t T = (local + ti - 1) / ti;
                if (T > nblocks && T % nblocks != 0) {
                    const int64_t bulk = (T / nblocks) * nblocks * ti;
                    const int64_t tail = local - bulk;
                    int g2 = d.glog;
                    const int minc = d.K <= 64 ? kTailSmallKMinC : kTailMinC;
                    while (g2 < 5 && (minc << (g2 + 1)) <= d.K && tail * (int64_t(2) << g2) <= (int64_t)nblocks * 256) ++g2;
                    if (g2 > d.glog) { bulk_end = runs[0].first + bulk; tail_glog = g2; }
                }
            }
            for (auto& r : runs)
                for (int64_t a = r.first; a < r.second;) {
                    const bool tail = bulk_end >= 0 && a >= bulk_end;
                    const int64_t len = tail ? (256 >> tail_glog) : ti;
                    all.push_back({q, i, a, std::min(r.second, a + len), tail ? tail_glog : 0});
                    a += len;
                }
        }
    }
    if (chunk_consumer)
        for (int c = 0; c < (int)chunk_consumer->size(); ++c)
            for (int q = 0; q < G; ++q) {
                all.push_back({q, n + (*chunk_consumer)[c], c, c + 1, 0});
            }
    const auto ttA = std::chrono::steady_clock::now();
    for (const GTask& t : all) ++toff[(size_t)t.vtx * G + t.rank + 1];
    for (size_t k = 1; k < toff.size(); ++k) toff[k] += toff[k - 1];
    tidx.resize(all.size());
    {
        std::vector<int32_t> fill(toff.begin(), toff.end() - 1);
        for (size_t t = 0; t < all.size(); ++t) tidx[fill[(size_t)all[t].vtx * G + all[t].rank]++] = (int32_t)t;
    }
    const auto ttB = std::chrono::steady_clock::now();
    // ---- broadcast flags (bit 0: T, bit 1: A)
    for (int j = 0; j < n; ++j) {
        VertexDesc& d = vd[j];
        d.bcast = 0;
        if (!d.part) continue;
        const int p = P.parent[j];
        bool aligned = false;
        if (p >= 0 && vd[p].part) {
            const int top_p = P.dep[p][vd[p].m - 1];
            aligned = std::find(P.dep[j].begin(), P.dep[j].end(), top_p) != P.dep[j].end();
        }
        d.bcast = (aligned ? 0 : 1) | 2;
    }
    // ---- pending counters per (rank, vertex): tasks each rank's copy of p waits for
    auto waits_on = [&](int p, int q) -> int64_t {
        int64_t s = 0;
        for (int j : P.children[p]) {
            if (vd[j].bcast & 1)
                for (int r = 0; r < G; ++r) s += (int64_t)tasks_of(j, r).size();
            else
                s += (int64_t)tasks_of(j, q).size();
        }
        return s;
    };
    std::vector<std::vector<int64_t>> pend(G, std::vector<int64_t>(n));
    for (int q = 0; q < G; ++q)
        for (int p = 0; p < n; ++p) pend[q][p] = waits_on(p, q) + (nv > n ? (int64_t)tasks_of(n + p, q).size() : 0);
    out.pending.assign(n, 0);
    for (int p = 0; p < n; ++p) {
        if (pend[rank][p] > INT32_MAX) { err = "internal: pending counter overflow"; return PASE_ERR_RESOURCE; }
        out.pending[p] = (int32_t)pend[rank][p];
    }
    const auto ttC = std::chrono::steady_clock::now();
    // ---- global list schedule: per-rank pools of nblocks CTAs, critical path first.
    // Estimated task time: ~3 us dependent-latency overhead + candidates at ~3e9/s per CTA.
    const int64_t ntk = (int64_t)all.size();
    std::vector<double> tdur(ntk), bl(nv, 0.0);
    const DurModel& dm = dur_model();
    for (int64_t t = 0; t < ntk; ++t) {
        if (all[t].vtx >= n) { tdur[t] = 4.0; continue; }  // a cost-table chunk
        const VertexDesc& d = vd[all[t].vtx];
        const double outs = d.shape < 0 ? 1 : cta_shape(d.shape) ? (double)d.cb1 * d.cb2 : d.q2 >= 0 ? kTile1 * kTile2 : kTile;
        double cand = (double)(all[t].i1 - all[t].i0) * d.K * outs;   // G1 items: kTile outputs too
        const double lanes = all[t].glog > 0 ? (double)(1 << (all[t].glog - d.glog)) : 1.0;   // wave tail
        const int f = dur_family(d);
        tdur[t] = dm.a[f] + cand / (dm.rate[f] * lanes);
    }
    // A/B only (PASE_DUR_FILE): measured per-task durations (us, float64 per task in task-id
    // order, e.g. from a PASE_TRACE timeline of the same plan) replace the model
    if (const char* df = std::getenv("PASE_DUR_FILE")) {
        if (FILE* fp = std::fopen(df, "rb")) {
            std::vector<double> m((size_t)ntk);
            if (std::fread(m.data(), sizeof(double), m.size(), fp) == m.size())
                for (int64_t t = 0; t < ntk; ++t)
                    if (all[t].vtx < n && m[t] > 0) tdur[t] = m[t];
            std::fclose(fp);
        }
    }
    std::vector<double> vtime(n, 0.0);
    for (int i = n - 1; i >= 0; --i) {                 // parents have higher ranks
        double work = 0.0, longest = 0.0;
        for (int q = 0; q < G; ++q)
            for (int32_t t : tasks_of(i, q)) { work += tdur[t]; longest = std::max(longest, tdur[t]); }
        vtime[i] = std::max(longest, work / ((double)nblocks * G));
        bl[i] = vtime[i] + (P.parent[i] >= 0 ? bl[P.parent[i]] : 0.0);
    }
    for (int i = n; i < nv; ++i) bl[i] = 4.0 + bl[i - n];
    const auto tt1 = std::chrono::steady_clock::now();
    std::vector<double> start(ntk, -1.0);
    std::vector<int32_t> start_seq;                     // tasks in simulated start order
    start_seq.reserve((size_t)ntk);
    if (!simulate) {
        // ready-queue claiming (single GPU): the order only ranks the leaves' tasks published at
        // the start -- critical path (bottom level) first; no list-schedule simulation
        for (int64_t t = 0; t < ntk; ++t) start[t] = -bl[all[t].vtx];
    } else {
        // ready (vertex, rank) runs: all tasks of a vertex share its priority, so the heap holds
        // one entry per released run and a cursor walks the run's tasks
        using RT = std::pair<double, int32_t>;                         // (priority, -(v*G+q))
        std::vector<std::priority_queue<RT>> ready(G);
        std::vector<int32_t> cursor((size_t)nv * G, 0);
        // an event finishes k equal-length tasks of one run started at the same time
        struct EV { double t; int32_t vq, k; bool operator>(const EV& o) const { return t != o.t ? t > o.t : vq > o.vq; } };
        std::priority_queue<EV, std::vector<EV>, std::greater<EV>> events;
        auto release = [&](int v, int q) {
            if (!tasks_of(v, q).empty()) ready[q].push({bl[v], -(v * G + q)});
        };
        for (int i = 0; i < nv; ++i)
            for (int q = 0; q < G; ++q)
                if (i >= n || pend[q][i] == 0) release(i, q);
        std::vector<int> free_w(G, nblocks);
        double now = 0.0;
        int64_t started = 0;
        while (started < ntk) {
            for (int q = 0; q < G; ++q)
                while (free_w[q] > 0 && !ready[q].empty()) {
                    const int32_t vq = -ready[q].top().second;
                    const Span run = tasks_of(vq / G, q);
                    const double d = tdur[run[cursor[vq]]];
                    int32_t k = 0;
                    while (k < free_w[q] && cursor[vq] < (int32_t)run.size() && tdur[run[cursor[vq]]] == d) {
                        start_seq.push_back(run[cursor[vq]]);
                        start[run[cursor[vq]++]] = now;
                        ++k;
                    }
                    if (cursor[vq] == (int32_t)run.size()) ready[q].pop();
                    started += k;
                    free_w[q] -= k;
                    events.push({now + d, vq, k});
                }
            if (started == ntk) break;
            if (events.empty()) { err = "internal: task DAG is not schedulable"; return PASE_ERR_STATE; }
            const EV e = events.top();
            events.pop();
            now = e.t;
            const int v = e.vq / G, q0 = e.vq % G;
            free_w[q0] += e.k;
            if (v >= n) {                               // cost chunks of vertex v - n done
                if ((pend[q0][v - n] -= e.k) == 0) release(v - n, q0);
                continue;
            }
            const int par = P.parent[v];
            if (par < 0) continue;
            if (vd[v].bcast & 1) {
                for (int q = 0; q < G; ++q)
                    if ((pend[q][par] -= e.k) == 0) release(par, q);
            } else if ((pend[q0][par] -= e.k) == 0) {
                release(par, q0);
            }
        }
    }
    const auto tt2 = std::chrono::steady_clock::now();
    // ---- this rank's tasks in simulated start order
    std::vector<int32_t> mine;
    mine.reserve((size_t)ntk);
    if (simulate) {                                     // start order; equal start times by task id
        for (int32_t t : start_seq)                    // ties: the simulation's priority order
            if (all[t].rank == rank) mine.push_back(t);
    } else {
        for (int64_t t = 0; t < ntk; ++t)
            if (all[t].rank == rank) mine.push_back((int32_t)t);
        std::stable_sort(mine.begin(), mine.end(), [&](int32_t a, int32_t b) { return start[a] < start[b]; });
    }
    out.tasks.clear();
    out.order.clear();
    std::vector<int32_t> local_id(ntk, -1);       // local ids in vertex order
    for (int i = 0; i < n; ++i) {
        vd[i].task0 = (int32_t)out.tasks.size();
        for (int32_t t : tasks_of(i, rank)) {
            local_id[t] = (int32_t)out.tasks.size();
            out.tasks.push_back({i, all[t].glog, all[t].i0, all[t].i1});
        }
        vd[i].ntasks = (int32_t)tasks_of(i, rank).size();
    }
    for (int i = n; i < nv; ++i)                        // cost-table tasks: vtx = -1 - chunk
        for (int32_t t : tasks_of(i, rank)) {
            local_id[t] = (int32_t)out.tasks.size();
            out.tasks.push_back({(int32_t)(-1 - all[t].i0), 0, 0, 0});
        }
    for (int32_t t : mine) out.order.push_back(local_id[t]);
    out.ready0.clear();                                 // leaves, in the static order's priority
    for (int32_t t : out.order)
        if (out.tasks[t].vtx >= 0 && out.pending[out.tasks[t].vtx] == 0) out.ready0.push_back(t);
    out.total_tasks = ntk;
    if (const char* tv = std::getenv("PASE_TIMING"); tv && tv[0] == '1')
        std::fprintf(stderr, "[pase] schedule: tasks+pending %.3f ms (build %.3f, sort %.3f, flags+pending %.3f, durations %.3f), list-schedule %.3f ms, order %.3f ms (%lld tasks)\n",
                     std::chrono::duration<double, std::milli>(tt1 - tt0).count(),
                     std::chrono::duration<double, std::milli>(ttA - tt0).count(),
                     std::chrono::duration<double, std::milli>(ttB - ttA).count(),
                     std::chrono::duration<double, std::milli>(ttC - ttB).count(),
                     std::chrono::duration<double, std::milli>(tt1 - ttC).count(),
                     std::chrono::duration<double, std::milli>(tt2 - tt1).count(),
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tt2).count(),
                     (long long)ntk);
    return PASE_OK;
}

}  // namespace pase
