// osim_harness.cuh -- the proxy-thread scenario harness on the GPU (SURVEY.md
// 8(f) row f3): workload._run_heuristic_schedule
// (/root/reference/pkg/src/offsim/workload.py:197-256), one thread per
// independent scenario.  A worker's next task becomes available when its
// previous task completes; the proxy forms a group from all available
// workers once the last HtD of the current group has gone through the DMA
// engine, reorders it with Algorithm 1 (heuristic.py:105-125, thread-level
// here) and appends it behind the commands still in flight (an incremental
// DeviceSim: every submit appends to the same FIFOs, engine.py:115-156).
// General path (null stages, IEEE division): bit-identical to the oracle.
#pragma once

#include "osim_deps.cuh"

namespace osim {

// Algorithm 1 for one group of m <= 16 tasks, in one thread.  td: the group's
// durations kind-major [3][16]; idr: id ranks within the group.  out: order.
template <int DMA>
__device__ void reorder_thread(const double* td, const uint8_t* idr, int m, double sigma, int sum_mode, int* out) {
    const Durs D{td, td, 1};
    unsigned nH = 0, nK = 0, nD = 0;
    for (int t = 0; t < m; ++t) {
        if (!(td[t] > 0.0)) nH |= 1u << t;
        if (!(td[kStride + t] > 0.0)) nK |= 1u << t;
        if (!(td[2 * kStride + t] > 0.0)) nD |= 1u << t;
    }
    auto sim = [&](uint64_t seq, int len, double& kEnd, double& idleK) {
        Sim<DMA, false, false, true> s;
        s.init(D, seq, len, sigma, 1.0, nH, nK, nD);
        s.run();
        kEnd = s.kEnd;
        idleK = s.idleK;
        return s.now;
    };
    if (m == 1) { out[0] = 0; return; }
    uint64_t ot = 0;
    int k = 0;
    unsigned rmask = (1u << m) - 1u;
    if (m >= 3) {  // select_first_task (heuristic.py:22-31)
        int best = -1;
        double b1 = 0, b2 = 0;
        for (int t = 0; t < m; ++t) {
            const double k1 = -__dsub_rn(td[kStride + t], td[t]), k2 = -td[2 * kStride + t];
            bool less;
            if (best < 0) less = true;
            else if (k1 < b1) less = true;
            else if (b1 < k1) less = false;
            else if (k2 < b2) less = true;
            else if (b2 < k2) less = false;
            else less = idr[t] < idr[best];
            if (less) { best = t; b1 = k1; b2 = k2; }
        }
        ot = (uint64_t)best;
        k = 1;
        rmask &= ~(1u << best);
        while (__popc(rmask) > 2) {  // select_next_task (heuristic.py:52-78)
            int bc = -1;
            double be = 0, bi = 0;
            for (int c = 0; c < m; ++c) {
                if (!((rmask >> c) & 1u)) continue;
                double kEnd, idleK;
                const double ms = sim(ot | ((uint64_t)c << (4 * k)), k + 1, kEnd, idleK);
                PySum ps;
                ps.reset();
                double tail = 0.0;
                bool any = false;
                for (int t = 0; t < m; ++t) {  // rest in rt (input) order
                    if (t == c || !((rmask >> t) & 1u)) continue;
                    ps.add(td[kStride + t], sum_mode);
                    const double d = td[2 * kStride + t];
                    if (!any || d < tail) tail = d;
                    any = true;
                }
                const double bound = __dadd_rn(__dadd_rn(kEnd, ps.result(sum_mode)), tail);
                const double est = (bound > ms) ? bound : ms;
                bool less;
                if (bc < 0) less = true;
                else if (est < be) less = true;
                else if (be < est) less = false;
                else if (idleK < bi) less = true;
                else if (bi < idleK) less = false;
                else less = idr[c] < idr[bc];
                if (less) { bc = c; be = est; bi = idleK; }
            }
            ot |= (uint64_t)bc << (4 * k);
            ++k;
            rmask &= ~(1u << bc);
        }
    }
    // select_last_tasks (heuristic.py:81-102)
    int a = __ffs(rmask) - 1;
    int b = __ffs(rmask & ~(1u << a)) - 1;
    if (idr[b] < idr[a]) { const int x = a; a = b; b = x; }
    double ke, ik;
    const double m_ab = sim(ot | ((uint64_t)a << (4 * k)) | ((uint64_t)b << (4 * (k + 1))), k + 2, ke, ik);
    const double m_ba = sim(ot | ((uint64_t)b << (4 * k)) | ((uint64_t)a << (4 * (k + 1))), k + 2, ke, ik);
    bool ab;
    if (m_ab < m_ba) ab = true;
    else if (m_ba < m_ab) ab = false;
    else ab = !(td[2 * kStride + a] <= td[2 * kStride + b]);
    ot |= ((uint64_t)(ab ? a : b) << (4 * k)) | ((uint64_t)(ab ? b : a) << (4 * (k + 1)));
    for (int i = 0; i < m; ++i) out[i] = nib(ot, i);
}

template <int DMA>
__global__ void __launch_bounds__(128) k_harness(const double* __restrict__ durs, const uint8_t* __restrict__ id_rank,
                                                 uint64_t S, int T, int N, double sigma, int sum_mode,
                                                 double* __restrict__ ms_out, uint8_t* __restrict__ ng_out,
                                                 uint8_t* __restrict__ sizes_out, double* __restrict__ start_out,
                                                 double* __restrict__ end_out, int* __restrict__ err) {
    const uint64_t sc = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (sc >= S) return;
    const int n = T * N;
    double gd[3 * kStride];  // the scenario's task durations, kind-major (local memory)
    for (int t = 0; t < kStride; ++t)
        for (int k = 0; k < 3; ++k) gd[k * kStride + t] = t < n ? durs[(sc * n + t) * 3 + k] : 1.0;
    uint8_t gr[kStride];
    for (int t = 0; t < n; ++t) gr[t] = id_rank[sc * n + t];
    DepSim<DMA> s;
    s.init(Durs{gd, gd, 1}, sigma, 0, 0, 0, false, n);  // empty queues, null stages marked done
    int next_idx[kStride];
    for (int w = 0; w < T; ++w) next_idx[w] = 0;
    unsigned avail = (T >= 32) ? ~0u : ((1u << T) - 1u);
    bool polling = true;
    int watched = -1;  // XFER/HtD queue index of the group's last HtD
    int ng = 0;
    bool ok = true;
    auto submit_group = [&]() {  // workload.py:219-233
        int tg[kStride], m = 0;
        for (int w = 0; w < T; ++w)
            if ((avail >> w) & 1u) tg[m++] = w * N + next_idx[w]++;
        avail = 0;
        double td[3 * kStride];
        uint8_t tr[kStride];
        for (int i = 0; i < m; ++i) {
            for (int k = 0; k < 3; ++k) td[k * kStride + i] = gd[k * kStride + tg[i]];
            int r = 0;
            for (int j = 0; j < m; ++j) r += gr[tg[j]] < gr[tg[i]];
            tr[i] = (uint8_t)r;
        }
        int ord[kStride];
        reorder_thread<DMA>(td, tr, m, sigma, sum_mode, ord);
        watched = -1;
        for (int i = 0; i < m; ++i) {  // DeviceSim.submit (engine.py:125-156)
            const int u = tg[ord[i]];
            if (s.nonnull(0, u)) { watched = s.q[0].len; s.q[0].push(u, 0); ++s.ncmd; }
            if (s.nonnull(1, u)) { s.q[2].push(u, 0); ++s.ncmd; }
            if (DMA == 2 && s.nonnull(2, u)) { s.q[1].push(u, 0); ++s.ncmd; }
        }
        if (DMA == 1)
            for (int i = 0; i < m; ++i) {
                const int u = tg[ord[i]];
                if (s.nonnull(2, u)) { s.q[0].push(u, 1); ++s.ncmd; }
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
        const int kb[3] = {s.kk[0], s.kk[1], s.kk[2]};
        const int cb[3] = {s.ck[0], s.ck[1], s.ck[2]};
        if (!s.step(tl)) {
            bool remaining = false;
            for (int w = 0; w < T; ++w) remaining |= next_idx[w] < N;
            ok = !remaining && s.drained();
            break;
        }
        for (int l = 0; l < 3; ++l) {  // the step's finalized commands
            if (s.h[l] == hb[l]) continue;
            if (l == 0 && hb[0] == watched) polling = true;
            const int t = s.ck[l];
            (void)kb; (void)cb;
            if (s.finished(t)) {
                const int w = t / N, j = t % N;
                if (j + 1 < N) avail |= 1u << w;
            }
        }
    }
    if (!ok) atomicExch(err, OSIM_ESTALL);
    ms_out[sc] = s.now;
    ng_out[sc] = (uint8_t)ng;
}

}  // namespace osim
