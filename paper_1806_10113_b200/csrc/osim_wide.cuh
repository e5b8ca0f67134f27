// osim_wide.cuh -- groups of 17..64 tasks on the general path.
//
// The reference's simulator, sampled search, heuristic and NoReorder
// sequences accept task groups of any size (engine.py:252-263,
// oracle.py:127-135, heuristic.py:105-125, workload.py:277-304); the packed
// 4-bit kernels stop at 16 tasks.  WideSim is DepSim (osim_deps.cuh) with
// byte-per-slot lane FIFOs and 64-bit done masks: the FIFOs are built the
// way DeviceSim.submit builds them (engine.py:115-156; null stages skipped,
// one submit per 1-DMA wave when `waves`), readiness is engine.py:165-178
// with the optional deps gate (:169-171), and each step is the reference's
// op sequence with IEEE division (:182-232), so every time is bit-identical
// to the oracle's.  TRACK adds k_end and idle["K"] for the heuristic
// (heuristic.py:46, :74; idle_report over K spans, which the K FIFO visits in
// sorted order).  One simulation per thread; these paths exist for
// coverage, not for the benchmark configs (all of which have n <= 16).
#pragma once

#include "osim_kernels.cuh"

namespace osim {

constexpr int kWideMax = 64;
constexpr int kWideBlock = 64;

template <int DMA, bool TRACK>
struct WideSim {
    const double* d;  // durations d[3 * task + kind] (the host layout)
    double sigma;
    const int8_t* dep;  // prerequisite task per task (-1 none), or nullptr
    uint8_t q[3][2 * kWideMax];  // 2-DMA: 0 HtD, 1 DtH, 2 K;  1-DMA: 0 XFER (bit 7 = DtH), 2 K
    int len[3], h[3];
    bool run[3];
    int ct[3], kk[3];  // running command: task, kind (0 HtD, 1 K, 2 DtH)
    double rem[3], nd[3];
    double now;
    uint64_t doneH, doneK, doneD;
    double kEnd, idleK;
    int kfin, ncmd;

    __device__ __forceinline__ double dur(int k, int t) const { return d[3 * t + k]; }
    __device__ __forceinline__ bool nonnull(int k, int t) const { return dur(k, t) > 0.0; }
    __device__ __forceinline__ int depof(int t) const { return dep ? (int)dep[t] : -1; }
    __device__ __forceinline__ void push(int l, int task, int isD) {
        OSIM_DCHECK(len[l] < 2 * kWideMax && task >= 0 && task < kWideMax);
        q[l][len[l]++] = (uint8_t)(task | (isD << 7));
    }

    // order: task ids of the len positions; ntask: tasks in the group
    __device__ void init(const double* dd, int ntask, double sg, const uint8_t* order, int n, const int8_t* dp,
                         bool waves) {
        d = dd;
        sigma = sg;
        dep = dp;
        now = 0.0;
        kEnd = 0.0;
        idleK = 0.0;
        kfin = 0;
        for (int l = 0; l < 3; ++l) { len[l] = 0; h[l] = 0; run[l] = false; rem[l] = 1.0; nd[l] = 1.0; }
        doneH = doneK = doneD = 0;
        for (int t = 0; t < ntask; ++t) {  // null stages are done from the start (engine.py:133-135)
            if (!nonnull(0, t)) doneH |= 1ull << t;
            if (!nonnull(1, t)) doneK |= 1ull << t;
            if (!nonnull(2, t)) doneD |= 1ull << t;
        }
        ncmd = 0;
        int w0 = 0;         // first position of the current wave
        uint64_t inw = 0;   // tasks of the current wave
        for (int p = 0; p <= n; ++p) {
            const int t = p < n ? order[p] : 0;
            const bool flush = p == n || (DMA == 1 && waves && depof(t) >= 0 && ((inw >> depof(t)) & 1ull));
            if (flush) {  // DeviceSim.submit of positions [w0, p)
                for (int i = w0; i < p; ++i) {
                    const int u = order[i];
                    if (nonnull(0, u)) { push(0, u, 0); ++ncmd; }
                    if (nonnull(1, u)) { push(2, u, 0); ++ncmd; }
                    if (nonnull(2, u) && DMA == 2) { push(1, u, 0); ++ncmd; }
                }
                if (DMA == 1)
                    for (int i = w0; i < p; ++i) {
                        const int u = order[i];
                        if (nonnull(2, u)) { push(0, u, 1); ++ncmd; }
                    }
                w0 = p;
                inw = 0;
            }
            if (p < n) inw |= 1ull << t;
        }
    }

    __device__ __forceinline__ bool finished(int t) const { return ((doneH & doneK & doneD) >> t) & 1ull; }
    __device__ __forceinline__ bool ready(int kind, int t) const {
        const int pd = depof(t);
        if (pd >= 0 && !finished(pd)) return false;  // engine.py:169-171
        if (kind == 1) return (doneH >> t) & 1ull;
        if (kind == 2) return ((doneK & doneH) >> t) & 1ull;
        return true;
    }
    __device__ __forceinline__ bool drained() const {
        return h[0] >= len[0] && h[1] >= len[1] && h[2] >= len[2];
    }

    // one DeviceSim.step(); false when nothing runs and nothing can start
    __device__ bool step(TimelineOut* tl) {
        for (int l = 0; l < 3; ++l) {  // start phase (engine.py:188-194)
            if (run[l] || h[l] >= len[l]) continue;
            const int e = q[l][h[l]], t = e & 0x7F;
            const int kind = (l == 2) ? 1 : ((l == 1) ? 2 : ((e & 0x80) ? 2 : 0));
            if (!ready(kind, t)) continue;
            run[l] = true;
            ct[l] = t;
            kk[l] = kind;
            nd[l] = dur(kind, t);
            rem[l] = nd[l];
            if constexpr (TRACK) {
                if (kind == 1 && kfin > 0 && now > kEnd) idleK = __dadd_rn(idleK, __dsub_rn(now, kEnd));
            }
            if (tl) tl->start[3 * t + kind] = now;
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
            const int t = ct[l];
            if (kk[l] == 0) doneH |= 1ull << t;
            else if (kk[l] == 1) doneK |= 1ull << t;
            else doneD |= 1ull << t;
            if constexpr (TRACK) {
                if (kk[l] == 1) { kEnd = now; ++kfin; }
            }
            if (tl) tl->end[3 * t + kk[l]] = now;
        }
        return true;
    }

    __device__ bool run_all(TimelineOut* tl = nullptr) {
        for (int s = 0; s < (ncmd + 1) * kSlowSteps && !drained(); ++s)
            if (!step(tl)) return false;
        return drained();
    }
};

// idle_report (engine.py:68-80) of a recorded timeline: per kind, spans
// sorted by (start, end), gaps accumulated left to right
__device__ inline void wide_idle(const double* start, const double* end, int n, double* res) {
    for (int k = 0; k < 3; ++k) {
        double idle = 0.0, prev_end = 0.0;
        uint64_t done = 0;
        for (int it = 0; it < n; ++it) {  // selection in (start, end) order
            int best = -1;
            for (int t = 0; t < n; ++t) {
                const double st = start[3 * t + k];
                if (st < 0.0 || ((done >> t) & 1ull)) continue;
                if (best < 0 || st < start[3 * best + k] ||
                    (st == start[3 * best + k] && end[3 * t + k] < end[3 * best + k]))
                    best = t;
            }
            if (best < 0) break;
            const double st = start[3 * best + k];
            if (it > 0 && st > prev_end) idle = __dadd_rn(idle, __dsub_rn(st, prev_end));
            prev_end = end[3 * best + k];
            done |= 1ull << best;
        }
        res[1 + k] = idle;
    }
}

// engine.simulate(tasks, profile, deps) / simulate_sequence: one timeline
template <int DMA>
__global__ void k_wide_timeline(const double* __restrict__ durs, int n, double sigma, const uint8_t* __restrict__ order,
                                const int8_t* __restrict__ dep, int waves, double* start, double* end, double* res,
                                int* err) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    for (int i = 0; i < 3 * n; ++i) { start[i] = -1.0; end[i] = -1.0; }
    WideSim<DMA, false> s;
    s.init(durs, n, sigma, order, n, dep, waves != 0);
    TimelineOut tl{start, end};
    if (!s.run_all(&tl)) { *err = OSIM_ESTALL; return; }
    res[0] = s.now;
    wide_idle(start, end, n, res);
}

// explicit orderings (sampled exhaustive_search, oracle.py:127-135)
template <int DMA>
__global__ void __launch_bounds__(kWideBlock) k_wide_eval_perms(const double* __restrict__ durs, int n, double sigma,
                                                                const uint8_t* __restrict__ perms, uint64_t cnt,
                                                                double* __restrict__ ms_out, Part* __restrict__ parts,
                                                                int* __restrict__ err) {
    __shared__ double sd[3 * kWideMax];
    __shared__ Part sh[32];
    for (int i = threadIdx.x; i < 3 * n; i += blockDim.x) sd[i] = durs[i];
    __syncthreads();
    Part acc;
    part_init(acc);
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += stride) {
        WideSim<DMA, false> s;
        s.init(sd, n, sigma, perms + i * (uint64_t)n, n, nullptr, false);
        if (!s.run_all()) atomicExch(err, OSIM_ESTALL);
        part_add<true>(acc, s.now, i, -kBig);
        ms_out[i] = s.now;
    }
    acc = block_reduce(acc, sh);
    if (threadIdx.x == 0) parts[blockIdx.x] = acc;
}

// NoReorder label sequences (workload.py:277-304): task (w, j) = w*N + j,
// prerequisite (w, j-1), 1-DMA waves
template <int DMA>
__global__ void __launch_bounds__(kWideBlock) k_wide_eval_labels(const double* __restrict__ durs, int T, int N,
                                                                 double sigma, const uint8_t* __restrict__ labels,
                                                                 uint64_t cnt, Part* __restrict__ parts,
                                                                 double* __restrict__ ms_out, int* __restrict__ err) {
    __shared__ double sd[3 * kWideMax];
    __shared__ int8_t sdep[kWideMax];
    __shared__ Part sh[32];
    const int n = T * N;
    for (int i = threadIdx.x; i < 3 * n; i += blockDim.x) sd[i] = durs[i];
    for (int t = threadIdx.x; t < n; t += blockDim.x) sdep[t] = (int8_t)((t % N) ? t - 1 : -1);
    __syncthreads();
    Part acc;
    part_init(acc);
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += stride) {
        uint8_t order[kWideMax];
        int c[kWideMax];
        for (int w = 0; w < T; ++w) c[w] = 0;
        for (int p = 0; p < n; ++p) {
            const int w = labels[i * n + p];
            order[p] = (uint8_t)(w * N + c[w]++);
        }
        WideSim<DMA, false> s;
        s.init(sd, n, sigma, order, n, sdep, true);
        if (!s.run_all()) atomicExch(err, OSIM_ESTALL);
        part_add<true>(acc, s.now, i, -kBig);
        ms_out[i] = s.now;
    }
    acc = block_reduce(acc, sh);
    if (threadIdx.x == 0) parts[blockIdx.x] = acc;
}

// Algorithm 1 (heuristic.py:105-125) in one thread, every candidate
// simulated from time 0 (select_first_task :22-31, select_next_task :52-78,
// _completion_estimate :34-49 with CPython's sum, select_last_tasks :81-102).
// gd: the group's durations [n][3]; idr: id ranks; ot: the order out.
// Returns the makespan of the chosen order (simulate(order)).
template <int DMA>
__device__ double wide_reorder(const double* gd, const uint8_t* idr, int n, double sigma, int sum_mode, uint8_t* ot,
                               bool& ok) {
    auto dur = [&](int k, int t) { return gd[3 * t + k]; };
    int k = 0;
    uint64_t rt = (n >= 64) ? ~0ull : ((1ull << n) - 1ull);
    if (n >= 3) {  // select_first_task: min of (-(t_k - t_htd), -t_dth, id)
        int best = -1;
        double b1 = 0, b2 = 0;
        for (int t = 0; t < n; ++t) {
            const double k1 = -__dsub_rn(dur(1, t), dur(0, t));
            const double k2 = -dur(2, t);
            bool less;
            if (best < 0) less = true;
            else if (k1 < b1) less = true;
            else if (b1 < k1) less = false;
            else if (k2 < b2) less = true;
            else if (b2 < k2) less = false;
            else less = idr[t] < idr[best];
            if (less) { best = t; b1 = k1; b2 = k2; }
        }
        ot[k++] = (uint8_t)best;
        rt &= ~(1ull << best);
    }
    while (__popcll(rt) > 2) {  // heuristic.py:120-123
        int bc = -1;
        double be = 0, bd = 0;
        for (uint64_t cm = rt; cm; cm &= cm - 1) {
            const int c = __ffsll((long long)cm) - 1;
            ot[k] = (uint8_t)c;
            WideSim<DMA, true> s;
            s.init(gd, n, sigma, ot, k + 1, nullptr, false);
            ok = s.run_all() && ok;
            // _completion_estimate: rest = rt minus c in rt (input) order
            PySum ps;
            ps.reset();
            double tail = 0.0;
            bool any = false;
            for (uint64_t r = rt & ~(1ull << c); r; r &= r - 1) {
                const int t = __ffsll((long long)r) - 1;
                ps.add(dur(1, t), sum_mode);
                const double x = dur(2, t);
                if (!any || x < tail) tail = x;
                any = true;
            }
            const double bound = __dadd_rn(__dadd_rn(s.kEnd, ps.result(sum_mode)), tail);
            const double est = (bound > s.now) ? bound : s.now;
            bool less;
            if (bc < 0) less = true;
            else if (est < be) less = true;
            else if (be < est) less = false;
            else if (s.idleK < bd) less = true;
            else if (bd < s.idleK) less = false;
            else less = idr[c] < idr[bc];
            if (less) { bc = c; be = est; bd = s.idleK; }
        }
        ot[k++] = (uint8_t)bc;
        rt &= ~(1ull << bc);
    }
    if (n >= 2) {  // select_last_tasks: the pair in id order, both orders simulated
        int a = __ffsll((long long)rt) - 1;
        int b = __ffsll((long long)(rt & (rt - 1))) - 1;
        if (idr[b] < idr[a]) { const int x = a; a = b; b = x; }
        double m2[2];
        for (int w = 0; w < 2; ++w) {
            ot[k] = (uint8_t)(w ? b : a);
            ot[k + 1] = (uint8_t)(w ? a : b);
            WideSim<DMA, false> s;
            s.init(gd, n, sigma, ot, n, nullptr, false);
            ok = s.run_all() && ok;
            m2[w] = s.now;
        }
        bool ab;
        if (m2[0] < m2[1]) ab = true;
        else if (m2[1] < m2[0]) ab = false;
        else ab = !(dur(2, a) <= dur(2, b));  // tie: shorter DtH last
        ot[k] = (uint8_t)(ab ? a : b);
        ot[k + 1] = (uint8_t)(ab ? b : a);
        return ab ? m2[0] : m2[1];
    }
    ot[0] = 0;  // reorder_batch returns [tg[0]] without simulating
    WideSim<DMA, false> s;
    s.init(gd, n, sigma, ot, 1, nullptr, false);
    ok = s.run_all() && ok;
    return s.now;
}

// reorder_batch over many groups, one group per thread
template <int DMA>
__global__ void __launch_bounds__(kWideBlock) k_wide_heuristic(const double* __restrict__ durs,
                                                               const uint8_t* __restrict__ id_rank, uint64_t B, int n,
                                                               double sigma, int sum_mode,
                                                               uint8_t* __restrict__ order_out,
                                                               double* __restrict__ ms_out,
                                                               uint32_t* __restrict__ nsims_out,
                                                               int* __restrict__ err) {
    const uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= B) return;
    uint8_t ot[kWideMax];
    bool ok = true;
    const double ms = wide_reorder<DMA>(durs + g * 3 * (uint64_t)n, id_rank + g * (uint64_t)n, n, sigma, sum_mode,
                                        ot, ok);
    if (!ok) atomicExch(err, OSIM_ESTALL);
    for (int p = 0; p < n; ++p) order_out[g * (uint64_t)n + p] = ot[p];
    ms_out[g] = ms;
    if (nsims_out) nsims_out[g] = (n >= 3) ? (uint32_t)(n * (n - 1) / 2 - 1) : (n == 2 ? 2u : 0u);
}

// The proxy-thread harness (workload.py:197-256) for
// scenarios of more than 16 tasks (the paper's T = 6, 8 workers x N = 4):
// k_harness (osim_harness.cuh) with WideSim FIFOs and 64-bit worker masks.
template <int DMA>
__global__ void __launch_bounds__(kWideBlock) k_wide_harness(const double* __restrict__ durs,
                                                             const uint8_t* __restrict__ id_rank, uint64_t S, int T,
                                                             int N, double sigma, int sum_mode,
                                                             double* __restrict__ ms_out, uint8_t* __restrict__ ng_out,
                                                             uint8_t* __restrict__ sizes_out,
                                                             double* __restrict__ start_out,
                                                             double* __restrict__ end_out, int* __restrict__ err) {
    const uint64_t sc = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (sc >= S) return;
    const int n = T * N;
    const double* gd = durs + sc * 3 * (uint64_t)n;
    const uint8_t* gr = id_rank + sc * (uint64_t)n;
    WideSim<DMA, false> s;
    s.init(gd, n, sigma, nullptr, 0, nullptr, false);  // empty FIFOs, null stages marked done
    int next_idx[kWideMax];
    for (int w = 0; w < T; ++w) next_idx[w] = 0;
    uint64_t avail = (T >= 64) ? ~0ull : ((1ull << T) - 1ull);
    bool polling = true;
    int watched = -1;  // XFER/HtD FIFO slot of the group's last HtD
    int ng = 0;
    bool ok = true;
    auto submit_group = [&]() {  // workload.py:219-233
        uint8_t tg[kWideMax];
        int m = 0;
        for (int w = 0; w < T; ++w)
            if ((avail >> w) & 1ull) tg[m++] = (uint8_t)(w * N + next_idx[w]++);
        avail = 0;
        double td[3 * kWideMax];
        uint8_t tr[kWideMax], ord[kWideMax];
        for (int i = 0; i < m; ++i) {
            for (int k = 0; k < 3; ++k) td[3 * i + k] = gd[3 * tg[i] + k];
            int r = 0;
            for (int j = 0; j < m; ++j) r += gr[tg[j]] < gr[tg[i]];
            tr[i] = (uint8_t)r;
        }
        wide_reorder<DMA>(td, tr, m, sigma, sum_mode, ord, ok);
        watched = -1;
        for (int i = 0; i < m; ++i) {  // DeviceSim.submit (engine.py:125-156)
            const int u = tg[ord[i]];
            if (s.nonnull(0, u)) { watched = s.len[0]; s.push(0, u, 0); ++s.ncmd; }
            if (s.nonnull(1, u)) { s.push(2, u, 0); ++s.ncmd; }
            if (DMA == 2 && s.nonnull(2, u)) { s.push(1, u, 0); ++s.ncmd; }
        }
        if (DMA == 1)
            for (int i = 0; i < m; ++i) {
                const int u = tg[ord[i]];
                if (s.nonnull(2, u)) { s.push(0, u, 1); ++s.ncmd; }
            }
        OSIM_DCHECK(ng < n && m >= 1);
        if (sizes_out) sizes_out[sc * n + ng] = (uint8_t)m;
        ++ng;
        polling = watched < 0;
    };
    TimelineOut tlo{start_out ? start_out + sc * 3 * n : nullptr, end_out ? end_out + sc * 3 * n : nullptr};
    TimelineOut* tl = start_out && end_out ? &tlo : nullptr;
    if (tl)
        for (int i = 0; i < 3 * n; ++i) { tl->start[i] = -1.0; tl->end[i] = -1.0; }
    submit_group();
    for (int guard = 0; guard < (3 * n + 1) * kSlowSteps + n + 1; ++guard) {
        if (polling && avail) submit_group();
        int hb[3];
        for (int l = 0; l < 3; ++l) hb[l] = s.h[l];
        if (!s.step(tl)) {
            bool remaining = false;
            for (int w = 0; w < T; ++w) remaining |= next_idx[w] < N;
            ok = ok && !remaining && s.drained();
            break;
        }
        for (int l = 0; l < 3; ++l) {  // the step's finalized commands
            if (s.h[l] == hb[l]) continue;
            if (l == 0 && hb[0] == watched) polling = true;
            const int t = s.ct[l];
            if (s.finished(t)) {
                const int w = t / N, j = t % N;
                if (j + 1 < N) avail |= 1ull << w;
            }
        }
    }
    if (!ok) atomicExch(err, OSIM_ESTALL);
    ms_out[sc] = s.now;
    ng_out[sc] = (uint8_t)ng;
}

}  // namespace osim
