// osim_big.cuh -- task groups of any size.
//
// The reference accepts groups of any size in simulate (engine.py:252-263,
// with deps and the 1-DMA waves of workload.simulate_sequence :277-304),
// sampled exhaustive_search (oracle.py:127-135), reorder_batch
// (heuristic.py:105-125), the proxy-thread harness (workload.py:197-256) and
// micro_simulate (oracle.py:60-95, _micro.py:19-143).  The register kernels
// stop at 16 tasks (4-bit positions) and WideSim at 64 (byte FIFOs, 64-bit
// masks).  BigSim is the same DeviceSim restatement with its three lane
// FIFOs (uint32 task ids) and per-task done bits in a per-simulation
// workspace in global memory, so n is bounded only by memory:
//   * FIFOs are built the way DeviceSim.submit builds them (engine.py:115-156:
//     null stages skipped, a 1-DMA submit appends the group's DtHs after its
//     HtDs, one submit per wave when `waves`);
//   * readiness is engine.py:165-178 with the optional deps gate (:169-171);
//   * every step is the reference's op sequence with IEEE division
//     (engine.py:182-232), so every time is bit-identical to the oracle's;
//   * idle_report (engine.py:68-80) is accumulated while the simulation runs:
//     a lane runs one command at a time, so a kind's commands start in FIFO
//     order, which is their (start, end) order, and the gap to the previous
//     command of the kind is added left to right exactly as the reference's
//     sorted loop adds it.
// These paths exist for coverage of the reference's API, not for the
// benchmark configs (all of which have n <= 16).
#pragma once

#include "osim_kernels.cuh"
#include "osim_micro.cuh"  // kMicroTol, kMicroBurst

namespace osim {

constexpr int kBigBlock = 128;
constexpr uint32_t kBigDtH = 0x80000000u;  // 1-DMA XFER FIFO entry: a DtH

// bytes of one simulation's workspace for n tasks: three FIFOs of 2n
// entries and one byte per task, 16-byte aligned
__host__ __device__ inline uint64_t big_ws_bytes(uint64_t n) { return (24ull * n + n + 15ull) & ~15ull; }

// Positions of a submitted list: a stored list, optionally followed by one
// or two more tasks (heuristic candidates: ot + [c], ot + [a, b]).
struct BigSeq {
    const uint32_t* a;
    uint64_t na;
    uint32_t x0, x1;
    int nx;
    __device__ __forceinline__ uint64_t size() const { return na + (uint64_t)nx; }
    __device__ __forceinline__ uint32_t operator()(uint64_t i) const { return i < na ? a[i] : (i == na ? x0 : x1); }
};

template <int DMA>
struct BigSim {
    const double* d;   // durations d[3 * task + kind] (kind 0 HtD, 1 K, 2 DtH)
    double sigma;
    const int32_t* dep;  // prerequisite task per task (-1 none), or nullptr
    uint32_t* q;         // lane l's FIFO at q[l * qcap]: 2-DMA 0 HtD, 1 DtH, 2 K; 1-DMA 0 XFER, 2 K
    uint64_t qcap;
    uint8_t* done;       // per task: bit 0 HtD, 1 K, 2 DtH finalized or null; bit 3 in the open submit wave
    uint64_t len[3], h[3];
    bool run[3];
    uint32_t ct[3];
    int kk[3];
    double rem[3], nd[3];
    double now;
    double idle[3], pend[3];  // idle_report per kind; end of the kind's latest command
    bool seen[3];
    uint64_t ncmd;
    int64_t last_htd;  // lane-0 slot of the latest submitted HtD (-1: none)

    __device__ __forceinline__ double dur(int k, uint32_t t) const { return d[3ull * t + k]; }
    __device__ __forceinline__ bool nonnull(int k, uint32_t t) const { return dur(k, t) > 0.0; }
    __device__ __forceinline__ int64_t depof(uint32_t t) const { return dep ? (int64_t)dep[t] : -1; }
    __device__ __forceinline__ void push(int l, uint32_t e) {
        OSIM_DCHECK(len[l] < qcap && (e & ~kBigDtH) < qcap / 2);
        q[(uint64_t)l * qcap + len[l]++] = e;
    }
    // k_end of heuristic.py:46: the latest K end, 0.0 without any K
    __device__ __forceinline__ double k_end() const { return seen[1] ? pend[1] : 0.0; }

    // empty queues over `ntask` tasks; null stages are done from the start
    // (engine.py:133-135)
    __device__ void begin(const double* dd, uint64_t ntask, double sg, const int32_t* dp, uint8_t* ws) {
        d = dd;
        sigma = sg;
        dep = dp;
        qcap = 2 * ntask;
        q = reinterpret_cast<uint32_t*>(ws);
        done = ws + 3 * qcap * sizeof(uint32_t);
        now = 0.0;
        ncmd = 0;
        last_htd = -1;
        for (int l = 0; l < 3; ++l) {
            len[l] = 0; h[l] = 0; run[l] = false; rem[l] = 1.0; nd[l] = 1.0;
            idle[l] = 0.0; pend[l] = 0.0; seen[l] = false;
        }
        for (uint64_t t = 0; t < ntask; ++t)
            done[t] = (uint8_t)((nonnull(0, (uint32_t)t) ? 0 : 1) | (nonnull(1, (uint32_t)t) ? 0 : 2) |
                                (nonnull(2, (uint32_t)t) ? 0 : 4));
    }

    // DeviceSim.submit of positions [a, b) of s (engine.py:125-156)
    __device__ void submit_range(const BigSeq& s, uint64_t a, uint64_t b) {
        for (uint64_t i = a; i < b; ++i) {
            const uint32_t u = s(i);
            if (nonnull(0, u)) { last_htd = (int64_t)len[0]; push(0, u); ++ncmd; }
            if (nonnull(1, u)) { push(2, u); ++ncmd; }
            if (DMA == 2 && nonnull(2, u)) { push(1, u); ++ncmd; }
        }
        if (DMA == 1)  // one-DMA launch order: the group's DtHs after its HtDs (:153-154)
            for (uint64_t i = a; i < b; ++i) {
                const uint32_t u = s(i);
                if (nonnull(2, u)) { push(0, u | kBigDtH); ++ncmd; }
            }
    }

    // one submit of the whole list, or (waves) one per wave: a task whose
    // prerequisite sits in the open wave starts a new one (workload.py:294-302)
    __device__ void submit(const BigSeq& s, bool waves) {
        const uint64_t cnt = s.size();
        if (!(DMA == 1 && waves)) { submit_range(s, 0, cnt); return; }
        uint64_t w0 = 0;
        for (uint64_t p = 0; p < cnt; ++p) {
            const uint32_t t = s(p);
            const int64_t pd = depof(t);
            if (pd >= 0 && (done[pd] & 8)) {
                submit_range(s, w0, p);
                for (uint64_t i = w0; i < p; ++i) done[s(i)] &= (uint8_t)~8u;
                w0 = p;
            }
            done[t] |= 8;
        }
        submit_range(s, w0, cnt);
        for (uint64_t i = w0; i < cnt; ++i) done[s(i)] &= (uint8_t)~8u;
    }

    __device__ __forceinline__ bool finished(uint32_t t) const { return (done[t] & 7) == 7; }
    __device__ __forceinline__ bool ready(int kind, uint32_t t) const {
        const int64_t pd = depof(t);
        if (pd >= 0 && !finished((uint32_t)pd)) return false;  // engine.py:169-171
        if (kind == 1) return done[t] & 1;                      // K: own HtD done
        if (kind == 2) return (done[t] & 3) == 3;               // DtH: own K and HtD done
        return true;
    }
    __device__ __forceinline__ bool drained() const { return h[0] >= len[0] && h[1] >= len[1] && h[2] >= len[2]; }

    // one DeviceSim.step(); false when nothing runs and nothing can start
    __device__ bool step(TimelineOut* tl) {
        for (int l = 0; l < 3; ++l) {  // start phase (engine.py:188-194)
            if (run[l] || h[l] >= len[l]) continue;
            OSIM_DCHECK(h[l] < len[l] && len[l] <= qcap);
            const uint32_t e = q[(uint64_t)l * qcap + h[l]], t = e & ~kBigDtH;
            const int kind = (l == 2) ? 1 : ((l == 1) ? 2 : ((e & kBigDtH) ? 2 : 0));
            if (!ready(kind, t)) continue;
            run[l] = true;
            ct[l] = t;
            kk[l] = kind;
            nd[l] = dur(kind, t);
            rem[l] = nd[l];
            if (seen[kind] && now > pend[kind]) idle[kind] = __dadd_rn(idle[kind], __dsub_rn(now, pend[kind]));
            if (tl) tl->start[3ull * t + kind] = now;
        }
        if (!run[0] && !run[1] && !run[2]) return false;
        const bool ov = DMA == 2 && run[0] && run[1];  // engine.py:200-204
        double rate[3];
        for (int l = 0; l < 3; ++l) rate[l] = (ov && l != 2) ? sigma : 1.0;  // :207-208
        double dt = 0.0;
        bool first = true;
        for (int l = 0; l < 3; ++l) {  // :210
            if (!run[l]) continue;
            const double v = __ddiv_rn(rem[l], rate[l]);
            if (first || v < dt) dt = v;
            first = false;
        }
        now = __dadd_rn(now, dt);  // :211
        for (int l = 0; l < 3; ++l) {  // :212-214
            if (!run[l]) continue;
            const double left = __dsub_rn(rem[l], __dmul_rn(dt, rate[l]));
            rem[l] = __dmul_rn(__ddiv_rn(pymax0(left), nd[l]), nd[l]);
        }
        for (int l = 0; l < 3; ++l) {  // finalize (:216-231)
            if (!run[l] || rem[l] > kEndEps) continue;
            run[l] = false;
            ++h[l];
            const uint32_t t = ct[l];
            const int k = kk[l];
            done[t] |= (uint8_t)(1u << k);
            pend[k] = now;
            seen[k] = true;
            if (tl) tl->end[3ull * t + k] = now;
        }
        return true;
    }

    __device__ bool run_all(TimelineOut* tl = nullptr) {
        for (uint64_t s = 0; s < (ncmd + 1) * kSlowSteps && !drained(); ++s)
            if (!step(tl)) return false;
        return drained();
    }
};

// ---- Algorithm 1 over a team of threads (a CTA, or one thread) ------------

struct BigKey {  // (estimate, idle_K, id) of heuristic.py:74, with the candidate's task and rt slot
    double est, idk;
    uint32_t idr, task;
    uint64_t slot;
    bool valid;
};

// (e, i, r) < (best): Python's tuple order on (float, float, id)
__device__ __forceinline__ bool big_less(const BigKey& a, const BigKey& b) {
    if (!b.valid) return a.valid;
    if (!a.valid) return false;
    if (a.est < b.est) return true;
    if (b.est < a.est) return false;
    if (a.idk < b.idk) return true;
    if (b.idk < a.idk) return false;
    return a.idr < b.idr;
}

struct BigTeamOne {
    __device__ __forceinline__ int rank() const { return 0; }
    __device__ __forceinline__ int size() const { return 1; }
    __device__ __forceinline__ void sync() const {}
    __device__ __forceinline__ BigKey argmin(const BigKey& k) const { return k; }
};

struct BigTeamCTA {
    BigKey* sh;  // [blockDim.x + 1] in shared memory
    __device__ __forceinline__ int rank() const { return threadIdx.x; }
    __device__ __forceinline__ int size() const { return blockDim.x; }
    __device__ __forceinline__ void sync() const { __syncthreads(); }
    __device__ BigKey argmin(const BigKey& k) const {
        sh[threadIdx.x] = k;
        __syncthreads();
        if (threadIdx.x == 0) {
            BigKey b = sh[0];
            for (int i = 1; i < (int)blockDim.x; ++i)
                if (big_less(sh[i], b)) b = sh[i];
            sh[blockDim.x] = b;
        }
        __syncthreads();
        const BigKey r = sh[blockDim.x];
        __syncthreads();
        return r;
    }
};

// reorder_batch (heuristic.py:105-125) of one group of n tasks: durations
// gd[n][3], id ranks idr[n] (Python string order of the ids); ot[n] gets the
// order, rt[n] is scratch (the remaining tasks in input order); ws: this
// thread's simulation workspace (big_ws_bytes(n)).  Candidates of a greedy
// round are spread over the team; every candidate is simulated from time 0
// (engine.simulate(ot + [cand])).  Returns simulate(order).makespan on
// rank 0.  select_first_task :22-31, select_next_task :52-78 with
// _completion_estimate :34-49 (CPython's sum over `rest` in rt order),
// select_last_tasks :81-102.
template <int DMA, class Team>
__device__ double big_reorder(const Team& tm, const double* gd, const uint32_t* idr, uint64_t n, double sigma,
                              int sum_mode, uint32_t* ot, uint32_t* rt, uint8_t* ws, bool& ok) {
    auto dur = [&](int k, uint64_t t) { return gd[3ull * t + k]; };
    const int me = tm.rank(), P = tm.size();
    if (me == 0)
        for (uint64_t t = 0; t < n; ++t) rt[t] = (uint32_t)t;
    tm.sync();
    uint64_t k = 0, m = n;
    if (n >= 3) {  // select_first_task: min of (-(t_k - t_htd), -t_dth, id)
        if (me == 0) {
            uint64_t best = 0;
            double b1 = 0.0, b2 = 0.0;
            for (uint64_t t = 0; t < n; ++t) {
                const double k1 = -__dsub_rn(dur(1, t), dur(0, t));
                const double k2 = -dur(2, t);
                bool less;
                if (t == 0) less = true;
                else if (k1 < b1) less = true;
                else if (b1 < k1) less = false;
                else if (k2 < b2) less = true;
                else if (b2 < k2) less = false;
                else less = idr[t] < idr[best];
                if (less) { best = t; b1 = k1; b2 = k2; }
            }
            ot[0] = (uint32_t)best;
            for (uint64_t j = best; j + 1 < n; ++j) rt[j] = rt[j + 1];  // rt.remove(first)
        }
        tm.sync();
        k = 1;
        m = n - 1;
    }
    while (m > 2) {  // heuristic.py:120-123
        BigKey best;
        best.valid = false;
        for (uint64_t j = (uint64_t)me; j < m; j += (uint64_t)P) {
            const uint32_t c = rt[j];
            BigSim<DMA> s;
            s.begin(gd, n, sigma, nullptr, ws);
            s.submit(BigSeq{ot, k, c, 0u, 1}, false);
            ok = s.run_all() && ok;
            PySum ps;  // rest = rt minus c, in rt (input) order
            ps.reset();
            double tail = 0.0;
            bool any = false;
            for (uint64_t r = 0; r < m; ++r) {
                if (r == j) continue;
                const uint32_t t = rt[r];
                ps.add(dur(1, t), sum_mode);
                const double x = dur(2, t);
                if (!any || x < tail) tail = x;
                any = true;
            }
            const double bound = __dadd_rn(__dadd_rn(s.k_end(), ps.result(sum_mode)), tail);
            BigKey key;
            key.est = (bound > s.now) ? bound : s.now;
            key.idk = s.idle[1];
            key.idr = idr[c];
            key.task = c;
            key.slot = j;
            key.valid = true;
            if (big_less(key, best)) best = key;
        }
        best = tm.argmin(best);
        if (me == 0) {
            OSIM_DCHECK(best.valid && best.slot < m && k < n);
            ot[k] = best.task;
            for (uint64_t j = best.slot; j + 1 < m; ++j) rt[j] = rt[j + 1];
        }
        tm.sync();
        ++k;
        --m;
    }
    double ms = 0.0;
    if (me == 0) {
        if (n >= 2) {  // select_last_tasks: the pair in id order, both completions simulated
            uint32_t a = rt[0], b = rt[1];
            if (idr[b] < idr[a]) { const uint32_t x = a; a = b; b = x; }
            double m2[2];
            for (int w = 0; w < 2; ++w) {
                BigSim<DMA> s;
                s.begin(gd, n, sigma, nullptr, ws);
                s.submit(BigSeq{ot, k, w ? b : a, w ? a : b, 2}, false);
                ok = s.run_all() && ok;
                m2[w] = s.now;
            }
            bool ab;
            if (m2[0] < m2[1]) ab = true;
            else if (m2[1] < m2[0]) ab = false;
            else ab = !(dur(2, a) <= dur(2, b));  // tie: (b, a) if dth_a <= dth_b
            ot[k] = ab ? a : b;
            ot[k + 1] = ab ? b : a;
            ms = ab ? m2[0] : m2[1];
        } else {  // n == 1: [tg[0]] (no simulation in the reference; the makespan is simulate([tg[0]]))
            ot[0] = 0;
            BigSim<DMA> s;
            s.begin(gd, n, sigma, nullptr, ws);
            s.submit(BigSeq{ot, 1, 0u, 0u, 0}, false);
            ok = s.run_all() && ok;
            ms = s.now;
        }
    }
    tm.sync();
    return ms;
}

__host__ __device__ inline uint32_t big_nsims(uint64_t n) {
    return n >= 3 ? (uint32_t)(n * (n - 1) / 2 - 1) : (n == 2 ? 2u : 0u);
}

// ---- kernels --------------------------------------------------------------

// engine.simulate(tasks, profile, deps) / simulate_sequence: one timeline;
// res = {makespan, idle HtD, idle K, idle DtH}
template <int DMA>
__global__ void k_big_timeline(const double* __restrict__ durs, uint64_t n, double sigma,
                               const uint32_t* __restrict__ order, const int32_t* __restrict__ dep, int waves,
                               uint8_t* ws, double* start, double* end, double* res, int* err) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    for (uint64_t i = 0; i < 3 * n; ++i) { start[i] = -1.0; end[i] = -1.0; }
    BigSim<DMA> s;
    s.begin(durs, n, sigma, dep, ws);
    s.submit(BigSeq{order, n, 0u, 0u, 0}, waves != 0);
    TimelineOut tl{start, end};
    if (!s.run_all(&tl)) { *err = OSIM_ESTALL; return; }
    res[0] = s.now;
    for (int k = 0; k < 3; ++k) res[1 + k] = s.idle[k];
}

// explicit orderings (sampled exhaustive_search, oracle.py:127-135);
// thread g uses the workspace ws + g * wsb
template <int DMA>
__global__ void __launch_bounds__(kBigBlock) k_big_eval_perms(const double* __restrict__ durs, uint64_t n,
                                                              double sigma, const uint32_t* __restrict__ perms,
                                                              uint64_t cnt, uint8_t* ws, uint64_t wsb,
                                                              double* __restrict__ ms_out, Part* __restrict__ parts,
                                                              int* __restrict__ err) {
    __shared__ Part sh[32];
    const uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint8_t* my = ws + g * wsb;
    Part acc;
    part_init(acc);
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = g; i < cnt; i += stride) {
        BigSim<DMA> s;
        s.begin(durs, n, sigma, nullptr, my);
        s.submit(BigSeq{perms + i * n, n, 0u, 0u, 0}, false);
        if (!s.run_all()) atomicExch(err, OSIM_ESTALL);
        part_add<true>(acc, s.now, i, -kBig);
        ms_out[i] = s.now;
    }
    acc = block_reduce(acc, sh);
    if (threadIdx.x == 0) parts[blockIdx.x] = acc;
}

// NoReorder label sequences (workload.py:277-327): task (w, j) = w*N + j,
// prerequisite dep[] = (w, j-1), 1-DMA waves; a thread's workspace holds its
// simulation, the label sequence's task order and T worker counters
template <int DMA>
__global__ void __launch_bounds__(kBigBlock) k_big_eval_labels(const double* __restrict__ durs, uint32_t T,
                                                               uint32_t N, double sigma,
                                                               const uint32_t* __restrict__ labels, uint64_t cnt,
                                                               const int32_t* __restrict__ dep, uint8_t* ws,
                                                               uint64_t wsb, double* __restrict__ ms_out,
                                                               Part* __restrict__ parts, int* __restrict__ err) {
    __shared__ Part sh[32];
    const uint64_t n = (uint64_t)T * N;
    const uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint8_t* my = ws + g * wsb;
    uint32_t* order = reinterpret_cast<uint32_t*>(my + big_ws_bytes(n));
    uint32_t* c = order + n;
    Part acc;
    part_init(acc);
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = g; i < cnt; i += stride) {
        for (uint32_t w = 0; w < T; ++w) c[w] = 0;
        for (uint64_t p = 0; p < n; ++p) {
            const uint32_t w = labels[i * n + p];
            order[p] = w * N + c[w]++;
        }
        BigSim<DMA> s;
        s.begin(durs, n, sigma, dep, my);
        s.submit(BigSeq{order, n, 0u, 0u, 0}, true);
        if (!s.run_all()) atomicExch(err, OSIM_ESTALL);
        part_add<true>(acc, s.now, i, -kBig);
        ms_out[i] = s.now;
    }
    acc = block_reduce(acc, sh);
    if (threadIdx.x == 0) parts[blockIdx.x] = acc;
}

// reorder_batch over many groups: one CTA per group (grid-stride), the
// candidates of each greedy round spread over the CTA's threads.  CTA b's
// workspace: ot[n], rt[n] (uint32), then one simulation workspace per thread.
__host__ __device__ inline uint64_t big_heur_cta_bytes(uint64_t n, int threads) {
    return ((8ull * n + 15ull) & ~15ull) + (uint64_t)threads * big_ws_bytes(n);
}

template <int DMA>
__global__ void __launch_bounds__(kBigBlock) k_big_heuristic(const double* __restrict__ durs,
                                                             const uint32_t* __restrict__ id_rank, uint64_t B,
                                                             uint64_t n, double sigma, int sum_mode, uint8_t* ws,
                                                             uint32_t* __restrict__ order_out,
                                                             double* __restrict__ ms_out,
                                                             uint32_t* __restrict__ nsims_out, int* __restrict__ err) {
    __shared__ BigKey sh[kBigBlock + 1];
    const BigTeamCTA tm{sh};
    uint8_t* cw = ws + (uint64_t)blockIdx.x * big_heur_cta_bytes(n, blockDim.x);
    uint32_t* ot = reinterpret_cast<uint32_t*>(cw);
    uint32_t* rt = ot + n;
    uint8_t* my = cw + ((8ull * n + 15ull) & ~15ull) + (uint64_t)threadIdx.x * big_ws_bytes(n);
    for (uint64_t g = blockIdx.x; g < B; g += gridDim.x) {
        bool ok = true;
        const double ms = big_reorder<DMA>(tm, durs + g * 3 * n, id_rank + g * n, n, sigma, sum_mode, ot, rt, my, ok);
        if (!ok) atomicExch(err, OSIM_ESTALL);
        for (uint64_t p = threadIdx.x; p < n; p += blockDim.x) order_out[g * n + p] = ot[p];
        if (threadIdx.x == 0) {
            ms_out[g] = ms;
            if (nsims_out) nsims_out[g] = big_nsims(n);
        }
        __syncthreads();  // ot / rt are rewritten for the next group
    }
}

// The proxy-thread harness (workload.py:197-256) for scenarios of any size:
// k_wide_harness's protocol with BigSim over the scenario's T*N tasks and the
// group reorder (groups of <= T tasks) in the same thread.
__host__ __device__ inline uint64_t big_harness_thread_bytes(uint64_t T, uint64_t N) {
    const uint64_t n = T * N;
    return big_ws_bytes(n) + big_ws_bytes(T) + ((24ull * T + 15ull) & ~15ull) /* td */ +
           ((4ull * T * 5ull + 15ull) & ~15ull) /* tg, tr, ord, rt, next */ + ((T + 15ull) & ~15ull) /* avail */;
}

template <int DMA>
__global__ void __launch_bounds__(kBigBlock) k_big_harness(const double* __restrict__ durs,
                                                           const uint32_t* __restrict__ id_rank, uint64_t S,
                                                           uint32_t T, uint32_t N, double sigma, int sum_mode,
                                                           uint8_t* ws, double* __restrict__ ms_out,
                                                           uint32_t* __restrict__ ng_out,
                                                           uint32_t* __restrict__ sizes_out,
                                                           double* __restrict__ start_out,
                                                           double* __restrict__ end_out, int* __restrict__ err) {
    const uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t n = (uint64_t)T * N;
    uint8_t* my = ws + g * big_harness_thread_bytes(T, N);
    uint8_t* sim_ws = my;
    uint8_t* grp_ws = sim_ws + big_ws_bytes(n);
    double* td = reinterpret_cast<double*>(grp_ws + big_ws_bytes(T));
    uint32_t* tg = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(td) + ((24ull * T + 15ull) & ~15ull));
    uint32_t* tr = tg + T;
    uint32_t* ord = tr + T;
    uint32_t* rtw = ord + T;
    uint32_t* next_idx = rtw + T;
    uint8_t* avail = reinterpret_cast<uint8_t*>(tg) + ((4ull * T * 5ull + 15ull) & ~15ull);
    const BigTeamOne one;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t sc = g; sc < S; sc += stride) {
        const double* gd = durs + sc * 3 * n;
        const uint32_t* gr = id_rank + sc * n;
        BigSim<DMA> s;
        s.begin(gd, n, sigma, nullptr, sim_ws);
        for (uint32_t w = 0; w < T; ++w) { next_idx[w] = 0; avail[w] = 1; }
        uint64_t navail = T;
        bool polling = true;
        int64_t watched = -1;  // lane-0 slot of the group's last HtD
        uint32_t ng = 0;
        bool ok = true;
        TimelineOut tlo{start_out ? start_out + sc * 3 * n : nullptr, end_out ? end_out + sc * 3 * n : nullptr};
        TimelineOut* tl = (start_out && end_out) ? &tlo : nullptr;
        if (tl)
            for (uint64_t i = 0; i < 3 * n; ++i) { tl->start[i] = -1.0; tl->end[i] = -1.0; }
        auto submit_group = [&]() {  // workload.py:219-233: sorted(available) workers' next tasks
            uint64_t m = 0;
            for (uint32_t w = 0; w < T; ++w)
                if (avail[w]) { tg[m++] = w * N + next_idx[w]++; avail[w] = 0; }
            navail = 0;
            for (uint64_t i = 0; i < m; ++i) {
                for (int k = 0; k < 3; ++k) td[3 * i + k] = gd[3ull * tg[i] + k];
                uint32_t r = 0;  // id ranks within the group
                for (uint64_t j = 0; j < m; ++j) r += gr[tg[j]] < gr[tg[i]];
                tr[i] = r;
            }
            big_reorder<DMA>(one, td, tr, m, sigma, sum_mode, ord, rtw, grp_ws, ok);
            for (uint64_t i = 0; i < m; ++i) ord[i] = tg[ord[i]];  // group positions -> scenario task ids
            s.last_htd = -1;
            s.submit(BigSeq{ord, m, 0u, 0u, 0}, false);  // DeviceSim.submit (engine.py:125-156)
            watched = s.last_htd;
            OSIM_DCHECK(ng < n && m >= 1 && m <= T);
            if (sizes_out) sizes_out[sc * n + ng] = (uint32_t)m;
            ++ng;
            polling = watched < 0;
        };
        submit_group();
        for (uint64_t guard = 0; guard < (3 * n + 1) * (uint64_t)kSlowSteps + n + 1; ++guard) {
            if (polling && navail) submit_group();
            uint64_t hb[3];
            for (int l = 0; l < 3; ++l) hb[l] = s.h[l];
            if (!s.step(tl)) {
                bool remaining = false;
                for (uint32_t w = 0; w < T; ++w) remaining |= next_idx[w] < N;
                ok = ok && !remaining && s.drained();
                break;
            }
            for (int l = 0; l < 3; ++l) {  // the step's finalized commands
                if (s.h[l] == hb[l]) continue;
                if (l == 0 && (int64_t)hb[0] == watched) polling = true;
                const uint32_t t = s.ct[l];
                if (s.finished(t)) {
                    const uint32_t w = t / N, j = t % N;
                    if (j + 1 < N && !avail[w]) { avail[w] = 1; ++navail; }
                }
            }
        }
        if (!ok) atomicExch(err, OSIM_ESTALL);
        ms_out[sc] = s.now;
        ng_out[sc] = ng;
    }
}

// micro_simulate (oracle.py:60-95, _micro.py:19-143) of one ordering of any
// size.  MicroSim (osim_micro.cuh) with positions instead of task masks: each
// queue is the ordering with that stage's nulls skipped, so a stage of the
// task at position p is done iff p lies before its queue head or the stage
// is null.
template <int DMA>
struct MicroBig {
    const double* d;
    const uint32_t* ord;
    uint64_t n;
    uint64_t hh, hd, hk;
    double rh, rd, rk, t, ms;
    long long step, ticks;

    __device__ __forceinline__ double dur(int k, uint64_t p) const { return d[3ull * ord[p] + k]; }
    __device__ __forceinline__ uint64_t skip(uint64_t p, int k) const {
        while (p < n && !(dur(k, p) > 0.0)) ++p;
        return p;
    }
    __device__ __forceinline__ bool done_h(uint64_t p) const { return p < hh || !(dur(0, p) > 0.0); }
    __device__ __forceinline__ bool done_k(uint64_t p) const { return p < hk || !(dur(1, p) > 0.0); }
    __device__ void init(const double* dd, const uint32_t* o, uint64_t nn) {
        d = dd; ord = o; n = nn;
        hh = skip(0, 0); hd = skip(0, 2); hk = skip(0, 1);
        rh = hh < n ? dur(0, hh) : 0.0;
        rd = hd < n ? dur(2, hd) : 0.0;
        rk = hk < n ? dur(1, hk) : 0.0;
        t = 0.0; ms = 0.0; step = 0; ticks = 0;
    }
    __device__ bool tick(double sigma, double dt, TimelineOut* tl) {
        const bool eh = hh < n;
        const bool ed = hd < n && (DMA == 2 || !eh) && done_k(hd) && done_h(hd);  // 1-DMA: DtHs after every HtD
        const bool ek = hk < n && done_h(hk);
        if (!eh && !ed && !ek) return false;
        const double rate = (DMA == 2 && eh && ed) ? sigma : 1.0;
        if (tl) {
            if (eh && tl->start[3ull * ord[hh] + 0] < 0.0) tl->start[3ull * ord[hh] + 0] = t;
            if (ed && tl->start[3ull * ord[hd] + 2] < 0.0) tl->start[3ull * ord[hd] + 2] = t;
            if (ek && tl->start[3ull * ord[hk] + 1] < 0.0) tl->start[3ull * ord[hk] + 1] = t;
        }
        // ticks up to the next finalization, as MicroSim::tick
        const double xt = __dmul_rn(dt, rate);
        const double big = 0x1p1000;
        double ah = eh ? rh : big, ad = ed ? rd : big, ak = ek ? rk : big;
        const double xh = eh ? xt : 0.0, xd = ed ? xt : 0.0, xk = ek ? dt : 0.0;
        long long k = 0;
        do {
            ah = __dsub_rn(ah, xh);
            ad = __dsub_rn(ad, xd);
            ak = __dsub_rn(ak, xk);
            ++k;
        } while (ah > kMicroTol && ad > kMicroTol && ak > kMicroTol && k < kMicroBurst);
        if (eh) rh = ah;
        if (ed) rd = ad;
        if (ek) rk = ak;
        step += k;
        ticks += k;
        t = __dmul_rn((double)step, dt);
        if (eh && rh <= kMicroTol) {
            if (tl) tl->end[3ull * ord[hh] + 0] = t;
            hh = skip(hh + 1, 0);
            if (hh < n) rh = dur(0, hh);
            ms = t;
        }
        if (ed && rd <= kMicroTol) {
            if (tl) tl->end[3ull * ord[hd] + 2] = t;
            hd = skip(hd + 1, 2);
            if (hd < n) rd = dur(2, hd);
            ms = t;
        }
        if (ek && rk <= kMicroTol) {
            if (tl) tl->end[3ull * ord[hk] + 1] = t;
            hk = skip(hk + 1, 1);
            if (hk < n) rk = dur(1, hk);
            ms = t;
        }
        return true;
    }
};

template <int DMA>
__global__ void k_big_micro_timeline(const double* __restrict__ durs, uint64_t n, double sigma, double dt,
                                     const uint32_t* __restrict__ order, long long max_ticks, double* start,
                                     double* end, double* res, int* err) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    for (uint64_t i = 0; i < 3 * n; ++i) { start[i] = -1.0; end[i] = -1.0; }
    MicroBig<DMA> s;
    s.init(durs, order, n);
    TimelineOut tl{start, end};
    while (s.tick(sigma, dt, &tl))
        if (s.ticks > max_ticks) { *err = OSIM_ESTALL; return; }
    res[0] = s.ms;
}

}  // namespace osim
