// osim_heur_lane.cuh -- Algorithm 1 (heuristic.py:105-125) with one task
// group per lane.
//
// k_heuristic_fast gives a warp 8 groups and spreads each greedy round's
// 8*m candidates over the 32 lanes: ceil(m/4) iterations leave 15 % of the
// lane slots empty, and the per-group serial phases (key argmin, checkpoint
// advance) run on 8 of 32 lanes.  Here every lane owns a group and walks its
// round's m candidates itself, kHLILP at a time (independent simulations
// interleaved in one instruction stream for ILP: with 13 warps per SM the
// kernel needs it to keep the issue slots busy), so only the last partial
// set of a round wastes slots and every serial phase runs on all 32 lanes.  The checkpoint of
// simulate(ot) (prefix sharing) lives in registers; the
// group's kernel and DtH durations live in shared memory in FastSim LAYOUT 6
// (nd and 1/nd arrays interleaved by lane, bank-conflict free), its HtD
// durations are read from global memory as a replay is set up (a replay
// starts at most two queued HtDs).  Shared memory per warp: 16 KB, so 13
// warps per SM (LAYOUT 2 with all three kinds: 24 KB, 9 warps).
// The per-candidate operation sequence is the one k_heuristic_fast runs
// (same FastSim steps from the same checkpoint, CPython's sum over `rest` in
// rt order, the (estimate, idle_K, id) key, select_last_tasks' tie rule), so
// orders, makespans and simulation counts are identical.
#pragma once

#include "osim_kernels.cuh"

namespace osim {

#ifndef OSIM_HL_W
#define OSIM_HL_W 1
#endif
// warps per CTA: one, so a finished warp's slot is refilled at once (the
// warps of a CTA are independent; a CTA's slot frees only when all finish)
constexpr int kHLW = OSIM_HL_W;
constexpr int kHLT = 32 * kHLW;                             // threads per CTA
#ifndef OSIM_HL_LPG
#define OSIM_HL_LPG 1
#endif
constexpr int kHLLPG = OSIM_HL_LPG;  // lanes per group (1: a group per lane; 2: lanes l, l + 16)
constexpr int kHLGPW = 32 / kHLLPG;  // groups per warp
#ifndef OSIM_HL_LAYOUT
#define OSIM_HL_LAYOUT 6
#endif
#ifndef OSIM_HL_HR
#define OSIM_HL_HR 1  // LAYOUT 6: {t_htd, 1/t_htd} pairs staged in global scratch
#endif
// FastSim layout: 2 (all three kinds in shared memory) or 6 (K and DtH in
// shared memory, a candidate's HtD durations loaded from global memory)
constexpr int kHLLay = kHLLPG == 1 ? OSIM_HL_LAYOUT : 3;
constexpr int kHLRows = kHLLay == 6 ? 32 : 48;  // shared rows per group
constexpr size_t kHLWarpSmem = 2 * kHLRows * kHLGPW * sizeof(double);  // nd + 1/nd, [rows][groups] each

#ifndef OSIM_HL_ILP
#define OSIM_HL_ILP 0  // 0: the measured best per DMA mode
#endif
// candidates per lane stepped together (2-DMA: 2, 1-DMA: 3 measured best)
template <int DMA>
__host__ __device__ constexpr int hl_ilp() {
    return OSIM_HL_ILP > 0 ? OSIM_HL_ILP : (kHLLPG == 2 ? (DMA == 2 ? 1 : 2) : (DMA == 2 ? 2 : 3));
}

#ifndef OSIM_HL_UNR
#define OSIM_HL_UNR 2
#endif
constexpr int kHLU = OSIM_HL_UNR;  // steps per phase test (warp vote)

// ILP simulations stepped in one loop (independent instruction streams):
// FastSim::run_phased for several candidates of a lane at once.
template <bool H0, int P, class FS>
__device__ __forceinline__ void run_multi(FS (&s)[P], int rest, double sigma, double rsig) {
    int st = 0;
    constexpr int DMA = FS::kDma;
    auto all_h = [&]() {
        bool d = true;
#pragma unroll
        for (int i = 0; i < P; ++i) d = d && s[i].s0 >= s[i].n4;
        return __all_sync(kFull, d);
    };
    auto all_k = [&]() {
        bool d = true;
#pragma unroll
        for (int i = 0; i < P; ++i) d = d && s[i].s2 >= s[i].n4;
        return __all_sync(kFull, d);
    };
    if constexpr (DMA == 2) {
#pragma unroll 1
        for (; st < rest; st += kHLU) {
            if (all_h()) break;
#pragma unroll
            for (int r = 0; r < kHLU; ++r)
#pragma unroll
                for (int i = 0; i < P; ++i) s[i].template step<H0>(sigma, rsig);
        }
#pragma unroll 1
        for (; st < rest; st += kHLU) {
            if (all_k()) break;
#pragma unroll
            for (int r = 0; r < kHLU; ++r)
#pragma unroll
                for (int i = 0; i < P; ++i) s[i].step_kd();
        }
#pragma unroll 1
        for (; st < rest; ++st)
#pragma unroll
            for (int i = 0; i < P; ++i) s[i].step_d();
    } else if constexpr (H0) {
#pragma unroll 1
        for (; st < rest; st += kHLU) {
            if (all_h()) break;
#pragma unroll
            for (int r = 0; r < kHLU; ++r)
#pragma unroll
                for (int i = 0; i < P; ++i) s[i].step(sigma, rsig);
        }
#pragma unroll 1
        for (; st < rest; st += kHLU) {
            if (all_k()) break;
#pragma unroll
            for (int r = 0; r < kHLU; ++r)
#pragma unroll
                for (int i = 0; i < P; ++i) s[i].step_1d();
        }
#pragma unroll 1
        for (; st < rest; ++st)
#pragma unroll
            for (int i = 0; i < P; ++i) s[i].step_1dd();
    } else {
#pragma unroll 1
        for (; st < rest; st += kHLU) {
            if (all_k()) break;
#pragma unroll
            for (int r = 0; r < kHLU; ++r)
#pragma unroll
                for (int i = 0; i < P; ++i) s[i].step_1dk();
        }
#pragma unroll 1
        for (; st < rest; ++st)
#pragma unroll
            for (int i = 0; i < P; ++i) s[i].step_1dd();
    }
}

template <int DMA, bool SP2>
__global__ void __launch_bounds__(kHLT) k_heuristic_lane(const double* __restrict__ durs,
                                                         const uint8_t* __restrict__ id_rank, uint64_t B, int n,
                                                         double sigma, int sum_mode,
                                                         uint8_t* __restrict__ order_out,
                                                         double* __restrict__ ms_out,
                                                         uint32_t* __restrict__ nsims_out,
                                                         const uint32_t* __restrict__ perm,
                                                         double2* __restrict__ hr) {
    using FS = FastSim<DMA, SP2, true, false, false, kHLLay>;
    constexpr bool kRH = kHLLay == 6;
    constexpr int kK0 = kRH ? 1 : 0;  // first kind held in shared memory
    constexpr int kHLILP = hl_ilp<DMA>();
    constexpr int W = kHLGPW;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane0 = threadIdx.x & 31;
    const int lane = lane0 % W;    // this lane's group within the warp
    const int sub = lane0 / W;     // which of the group's lanes (kHLLPG = 2: candidate sets alternate)
    double* nd = reinterpret_cast<double*>(smem_raw + warp * kHLWarpSmem);  // [48][W]
    double* rcp = nd + kHLRows * W;
    const uint64_t g0 = ((uint64_t)blockIdx.x * kHLW + warp) * W;
    if (g0 >= B) return;  // whole warp leaves together; no block barriers below
    const bool live = g0 + lane < B;
    // perm (nullable): the batch position this lane's group comes from (and
    // whose outputs it writes) -- groups ordered by heur_sort_keys so a warp's
    // 32 groups have similar replay lengths
    const uint64_t g = live ? (perm ? (uint64_t)perm[g0 + lane] : g0 + lane) : 0;
    const int Gv = (int)((B - g0) < (uint64_t)W ? (B - g0) : (uint64_t)W);
    // stage this lane's group: entry (kind k, task t) at [(k*16 + t)*32 + lane]
    // (bank-conflict-free stores; the strided loads hit L1 after the first
    // touch of each line); tasks >= n get 1.0
    (void)Gv;  // (tasks of a lane past the batch end are 1.0 placeholders)
    for (int kt = sub * (kHLRows / kHLLPG); kt < (sub + 1) * (kHLRows / kHLLPG); ++kt) {  // a group's lanes split it
        const int k = (kt >> 4) + kK0, t = kt & 15;
        const double v = (live && t < n) ? durs[g * 3 * (uint64_t)n + 3 * t + k] : 1.0;
        nd[kt * W + lane] = v;
        rcp[kt * W + lane] = __ddiv_rn(1.0, v);
    }
    __syncwarp();
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(nd) + 8u * (uint32_t)lane;
    auto DV = [&](int k, int t) { return nd[((k - kK0) * 16 + t) * W + lane]; };
    const double* gH = durs + g * 3 * (uint64_t)n;  // LAYOUT 6: HtD durations of task t at gH[3t]
    auto HV = [&](int t) { return kRH ? ((live && t < n) ? gH[3 * t] : 1.0) : DV(0, t); };
    // a candidate's HtD {nd, 1/nd}: from the staged pairs (hr), else loaded
    // and divided here
    double2* hrg = hr ? hr + g * 16 : nullptr;
    if (kRH && hrg && live) {
        for (int t = 0; t < n; ++t) {
            const double h = gH[3 * t];
            hrg[t] = make_double2(h, __ddiv_rn(1.0, h));
        }
    }
    auto HR = [&](int t) {
        if (hrg && live) return hrg[t];
        const double h = HV(t);
        return make_double2(h, __ddiv_rn(1.0, h));
    };
    uint64_t idr = 0;  // id rank per task, 4 bits each
    for (int t = 0; t < n; ++t) idr |= (uint64_t)(live ? id_rank[g * (uint64_t)n + t] : (uint8_t)t) << (4 * t);
    auto IR = [&](int t) { return (int)((idr >> (4 * t)) & 0xF); };
    const double rsig = __ddiv_rn(1.0, sigma);

    // select_first_task (heuristic.py:22-31) and the first checkpoint
    typename FS::Ck ck;
    uint64_t ot = 0, cand = 0;
    {
        const unsigned all = (1u << n) - 1u;
        unsigned rm = all;
        FS s;
        if (n >= 3) {
            int best = 0;
            double b1 = 0, b2 = 0;
            for (int t = 0; t < n; ++t) {
                const double k1 = -__dsub_rn(DV(1, t), HV(t));
                const double k2 = -DV(2, t);
                bool less;
                if (t == 0) less = true;
                else if (k1 < b1) less = true;
                else if (b1 < k1) less = false;
                else if (k2 < b2) less = true;
                else if (b2 < k2) less = false;
                else less = IR(t) < IR(best);
                if (less) { best = t; b1 = k1; b2 = k2; }
            }
            ot = (uint64_t)best;
            rm = all & ~(1u << best);
            s.init(base, ot, 1);
            if constexpr (kRH) { const double h = HV(best); s.set_htd(h, __ddiv_rn(1.0, h)); }
            for (int q = 0; q < 3 * kMaxN && s.htd_done() < 1; ++q) s.step(sigma, rsig);
        } else {
            s.init(base, 0, 1);  // empty prefix: the initial state
        }
        s.save(ck);
        for (int t = n - 1; t >= 0; --t)
            if ((rm >> t) & 1u) cand = (cand << 4) | (uint64_t)t;
    }

    const int k0 = (n >= 3) ? 1 : 0;
    for (int k = k0; n - k > 2; ++k) {  // heuristic.py:120-123
        const int m = n - k;
        FS c0;  // the checkpoint's finalized count fixes every candidate's replay bound
        c0.load(ck);
        const int rest = __reduce_max_sync(kFull, 3 * (k + 1) - c0.finalized());
        int bj = -1;
        double be = 0, bd = 0;
        int br = 0;
        for (int j0 = 0; j0 < m; j0 += kHLLPG * kHLILP) {
            const int j = j0 + sub * kHLILP;  // this lane's candidates j .. j + P - 1 (>= m: surplus)
            int cj[kHLILP], cc[kHLILP];
            FS sim[kHLILP];
#pragma unroll
            for (int i = 0; i < kHLILP; ++i) {
                cj[i] = (j + i < m) ? j + i : m - 1;  // a surplus slot repeats the last candidate
                cc[i] = rt_at(cand, cj[i]);
                sim[i].init(base, ot | ((uint64_t)cc[i] << (4 * k)), k + 1);
                sim[i].load(ck);
                if constexpr (kRH) { const double2 h = HR(cc[i]); sim[i].set_htd(h.x, h.y); }
                sim[i].start_htd();
            }
            run_multi<false>(sim, rest, sigma, rsig);
            // _completion_estimate (heuristic.py:34-49): CPython's sum of the
            // rest's t_k in rt order and min t_dth.  The set's candidates are
            // the rt slots j .. j+P-1 (a surplus one has virtual slot j+i >= m,
            // its result unused), so every rest shares the slots before j: their
            // running sum state is computed once and forked; inside [j, j+P)
            // each candidate skips its own slot (a warp-uniform test); after
            // it every candidate continues its own state, and the tail minimum
            // (order-free) over those slots is shared.
            double f[kHLILP], e[kHLILP], tl[kHLILP];
            auto nadd = [&](double& fs, double& es, double x) {
                const double t = __dadd_rn(fs, x);
                if (sum_mode) {  // Neumaier (CPython >= 3.12): TwoSum error of f + x
                    const double p = __dsub_rn(t, fs);
                    es = __dadd_rn(es, __dadd_rn(__dsub_rn(fs, __dsub_rn(t, p)), __dsub_rn(x, p)));
                }
                fs = t;
            };
            {
                double pf = 0.0, pe = 0.0, ptl = kBig;
                uint64_t rl = cand;
#pragma unroll 2
                for (int q = 0; q < j; ++q, rl >>= 4) {  // common prefix
                    const int u = (int)(rl & 0xF);
                    nadd(pf, pe, DV(1, u));
                    ptl = dmin(DV(2, u), ptl);
                }
#pragma unroll
                for (int i = 0; i < kHLILP; ++i) { f[i] = pf; e[i] = pe; tl[i] = ptl; }
#pragma unroll
                for (int q2 = 0; q2 < kHLILP; ++q2) {  // the set's own slots
                    if (j + q2 >= m) break;
                    const int u = (int)((rl >> (4 * q2)) & 0xF);
                    const double x = DV(1, u), y = DV(2, u);
#pragma unroll
                    for (int i = 0; i < kHLILP; ++i) {
                        if (i == q2) continue;
                        nadd(f[i], e[i], x);
                        tl[i] = dmin(y, tl[i]);
                    }
                }
                double stl = kBig;
                rl >>= 4 * kHLILP;
#pragma unroll 2
                for (int q = j + kHLILP; q < m; ++q, rl >>= 4) {  // common suffix, separate sums
                    const int u = (int)(rl & 0xF);
                    const double x = DV(1, u);
                    stl = dmin(DV(2, u), stl);
#pragma unroll
                    for (int i = 0; i < kHLILP; ++i) nadd(f[i], e[i], x);
                }
#pragma unroll
                for (int i = 0; i < kHLILP; ++i) tl[i] = dmin(stl, tl[i]);
            }
#pragma unroll
            for (int i = 0; i < kHLILP; ++i) {
                if (sum_mode && e[i] != 0.0 && isfinite(e[i])) f[i] = __dadd_rn(f[i], e[i]);
                const double bound = __dadd_rn(__dadd_rn(sim[i].kEnd, f[i]), tl[i]);
                const double est = (bound > sim[i].now) ? bound : sim[i].now;
                const int r = IR(cc[i]);
                if (j + i < m && (bj < 0 || key_less(est, sim[i].idleK, r, be, bd, br))) {
                    bj = cj[i]; be = est; bd = sim[i].idleK; br = r;
                }
            }
        }
        if constexpr (kHLLPG > 1) {  // the group's lanes exchange their best keys
#pragma unroll
            for (int off = W; off < 32; off <<= 1) {
                const int oj = __shfl_xor_sync(kFull, bj, off), orr = __shfl_xor_sync(kFull, br, off);
                const double oe = __shfl_xor_sync(kFull, be, off), od = __shfl_xor_sync(kFull, bd, off);
                if (oj >= 0 && (bj < 0 || key_less(oe, od, orr, be, bd, br))) { bj = oj; be = oe; bd = od; br = orr; }
            }
        }
        OSIM_DCHECK(bj >= 0 && bj < m);
        const int c = rt_at(cand, bj);
        ot |= (uint64_t)c << (4 * k);
        cand = rt_drop(cand, bj);
        // advance the checkpoint by the chosen task (prefix length k + 1)
        FS s;
        s.init(base, ot, k + 1);
        s.load(ck);
        if constexpr (kRH) { const double2 h = HR(c); s.set_htd(h.x, h.y); }
        s.start_htd();  // the chosen task's HtD, the queue's last
        if constexpr (DMA == 2) {
            for (int q = 0; q < 3 * kMaxN && s.htd_done() < k + 1; ++q) s.template step<false>(sigma, rsig);
        } else {
            for (int q = 0; q < 3 * kMaxN && s.htd_done() < k + 1; ++q) s.step_1dk();
        }
        s.save(ck);
    }

    const int kl = n - 2;  // select_last_tasks (heuristic.py:81-102)
    double ms;
    if (n >= 2) {
        int a = rt_at(cand, 0), b = rt_at(cand, 1);
        if (IR(b) < IR(a)) { const int x = a; a = b; b = x; }
        FS sp[2];
        sp[0].init(base, ot | ((uint64_t)a << (4 * kl)) | ((uint64_t)b << (4 * (kl + 1))), n);
        sp[1].init(base, ot | ((uint64_t)b << (4 * kl)) | ((uint64_t)a << (4 * (kl + 1))), n);
        sp[0].load(ck);
        sp[1].load(ck);
        if constexpr (kRH) {  // the two queued HtDs, in each ordering's order
            const double2 pa = HR(a), pb = HR(b);
            sp[0].set_htd(pa.x, pa.y, pb.x, pb.y);
            sp[1].set_htd(pb.x, pb.y, pa.x, pa.y);
        }
        const int rest = __reduce_max_sync(kFull, 3 * n - sp[0].finalized());
        run_multi<true>(sp, rest, sigma, rsig);
        const double m_ab = sp[0].now, m_ba = sp[1].now;
        bool ab;
        if (m_ab < m_ba) ab = true;
        else if (m_ba < m_ab) ab = false;
        else ab = !(DV(2, a) <= DV(2, b));  // tie: shorter DtH last
        ot |= ((uint64_t)(ab ? a : b) << (4 * kl)) | ((uint64_t)(ab ? b : a) << (4 * (kl + 1)));
        ms = ab ? m_ab : m_ba;  // simulate(ot + chosen pair)
    } else {
        FS s;  // n == 1: reorder_batch returns [tg[0]] without simulating
        s.init(base, 0, 1);
        if constexpr (kRH) { const double h = HV(0); s.set_htd(h, __ddiv_rn(1.0, h)); }
        for (int st = 0; st < 3; ++st) s.step(sigma, rsig);
        ms = s.now;
    }
    if (live && sub == 0) {
        ms_out[g] = ms;
        if (nsims_out) nsims_out[g] = (n >= 3) ? (uint32_t)(n * (n - 1) / 2 - 1) : (n == 2 ? 2u : 0u);
        for (int p = 0; p < n; ++p) order_out[g * (uint64_t)n + p] = (uint8_t)nib(ot, p);
    }
}

}  // namespace osim

namespace osim {

// Sort key of a group for k_heuristic_lane's warp assignment: its kernel
// share sum(t_k) / (sum(t_htd) + sum(t_dth)) in 1/64 steps up to 4 (8 bits).
// Kernel-heavy groups carry a long K/DtH backlog at every checkpoint
// (long candidate replays), transfer-heavy ones a short one; a warp's replay
// length is the longest of its 32 groups', so similar groups share warps.
// Only the assignment changes: every group's result is computed from its own
// data and written to its own position.
static __global__ void k_heur_sort_keys(const double* __restrict__ durs, uint64_t B, int n, uint8_t* __restrict__ key,
                                        uint32_t* __restrict__ idx) {
    const uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= B) return;
    const double* d = durs + g * 3 * (uint64_t)n;
    double h = 0.0, k = 0.0;
    for (int t = 0; t < n; ++t) {
        h += d[3 * t] + d[3 * t + 2];
        k += d[3 * t + 1];
    }
    const double q = h > 0.0 ? k / h * 64.0 : 255.0;
    key[g] = (uint8_t)(q < 255.0 ? q : 255.0);
    idx[g] = (uint32_t)g;
}

}  // namespace osim
