// osim_heur_lane.cuh -- Algorithm 1 (heuristic.py:105-125) with one task
// group per lane.
//
// k_heuristic_fast gives a warp 8 groups and spreads each greedy round's
// 8*m candidates over the 32 lanes: ceil(m/4) iterations leave 15 % of the
// lane slots empty, and the per-group serial phases (key argmin, checkpoint
// advance) run on 8 of 32 lanes.  Here every lane owns a group and walks its
// round's m candidates itself, two at a time (two independent simulations
// interleaved in one instruction stream for ILP), so only odd m wastes a
// slot (6 %) and every serial phase runs on all 32 lanes.  The checkpoint of
// simulate(ot) (prefix sharing) lives in registers; the
// group's durations live in shared memory in FastSim LAYOUT 2 (nd and 1/nd
// arrays interleaved by lane, bank-conflict free).  Shared memory per warp:
// 24 KB, so 9 warps per SM; the ILP makes up for the fewer warps.
// The per-candidate operation sequence is the one k_heuristic_fast runs
// (same FastSim steps from the same checkpoint, CPython's sum over `rest` in
// rt order, the (estimate, idle_K, id) key, select_last_tasks' tie rule), so
// orders, makespans and simulation counts are identical.
#pragma once

#include "osim_kernels.cuh"

namespace osim {

constexpr int kHLW = 3;                                     // warps per CTA
constexpr int kHLT = 32 * kHLW;                             // threads per CTA
constexpr size_t kHLWarpSmem = 2 * 48 * 32 * sizeof(double);  // nd + 1/nd, [48][32] each

// Two simulations stepped in one loop (independent instruction streams):
// FastSim::run_phased for a pair of lanes' worth of work.
template <bool H0, class FS>
__device__ __forceinline__ void run_pair(FS& a, FS& b, int rest, double sigma, double rsig) {
    int st = 0;
    constexpr int DMA = FS::kDma;
    if constexpr (DMA == 2) {
#pragma unroll 1
        for (; st < rest; st += 2) {
            if (__all_sync(kFull, a.s0 >= a.n4 && b.s0 >= b.n4)) break;
            a.template step<H0>(sigma, rsig);
            b.template step<H0>(sigma, rsig);
            a.template step<H0>(sigma, rsig);
            b.template step<H0>(sigma, rsig);
        }
#pragma unroll 1
        for (; st < rest; st += 2) {
            if (__all_sync(kFull, a.s2 >= a.n4 && b.s2 >= b.n4)) break;
            a.step_kd();
            b.step_kd();
            a.step_kd();
            b.step_kd();
        }
#pragma unroll 1
        for (; st < rest; ++st) {
            a.step_d();
            b.step_d();
        }
    } else if constexpr (H0) {
#pragma unroll 1
        for (; st < rest; st += 2) {
            if (__all_sync(kFull, a.s0 >= a.n4 && b.s0 >= b.n4)) break;
            a.step(sigma, rsig);
            b.step(sigma, rsig);
            a.step(sigma, rsig);
            b.step(sigma, rsig);
        }
#pragma unroll 1
        for (; st < rest; st += 2) {
            if (__all_sync(kFull, a.s2 >= a.n4 && b.s2 >= b.n4)) break;
            a.step_1d();
            b.step_1d();
            a.step_1d();
            b.step_1d();
        }
#pragma unroll 1
        for (; st < rest; ++st) {
            a.step_1dd();
            b.step_1dd();
        }
    } else {
#pragma unroll 1
        for (; st < rest; st += 2) {
            if (__all_sync(kFull, a.s2 >= a.n4 && b.s2 >= b.n4)) break;
            a.step_1dk();
            b.step_1dk();
            a.step_1dk();
            b.step_1dk();
        }
#pragma unroll 1
        for (; st < rest; ++st) {
            a.step_1dd();
            b.step_1dd();
        }
    }
}

template <int DMA, bool SP2>
__global__ void __launch_bounds__(kHLT) k_heuristic_lane(const double* __restrict__ durs,
                                                         const uint8_t* __restrict__ id_rank, uint64_t B, int n,
                                                         double sigma, int sum_mode,
                                                         uint8_t* __restrict__ order_out,
                                                         double* __restrict__ ms_out,
                                                         uint32_t* __restrict__ nsims_out) {
    using FS = FastSim<DMA, SP2, true, false, false, 2>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* nd = reinterpret_cast<double*>(smem_raw + warp * kHLWarpSmem);  // [48][32]
    double* rcp = nd + 48 * 32;
    const uint64_t g0 = ((uint64_t)blockIdx.x * kHLW + warp) * 32;
    if (g0 >= B) return;  // whole warp leaves together; no block barriers below
    const uint64_t g = g0 + lane;
    const bool live = g < B;
    const int Gv = (int)((B - g0) < 32 ? (B - g0) : 32);
    // stage the warp's groups (contiguous in HBM) with coalesced loads: entry
    // (kind k, task t) of lane gi at [(k*16 + t)*32 + gi]; tasks >= n get 1.0
    for (int e = lane; e < 48 * 32; e += 32) {
        const int gi = e / 48, r = e % 48, t = r / 3, k = r % 3;
        const int idx = (k * 16 + t) * 32 + gi;
        double v = 1.0;
        if (gi < Gv && t < n) v = durs[(g0 + gi) * 3 * (uint64_t)n + 3 * t + k];
        nd[idx] = v;  // every (k, t, gi) exactly once
        rcp[idx] = __ddiv_rn(1.0, v);
    }
    __syncwarp();
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(nd) + 8u * (uint32_t)lane;
    auto DV = [&](int k, int t) { return nd[(k * 16 + t) * 32 + lane]; };
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
                const double k1 = -__dsub_rn(DV(1, t), DV(0, t));
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
        for (int j = 0; j < m; j += 2) {
            const bool two = j + 1 < m;
            const int ja = j, jb = two ? j + 1 : j;
            const int ca = rt_at(cand, ja), cb = rt_at(cand, jb);
            FS sa, sb;
            sa.init(base, ot | ((uint64_t)ca << (4 * k)), k + 1);
            sb.init(base, ot | ((uint64_t)cb << (4 * k)), k + 1);
            sa.load(ck);
            sb.load(ck);
            sa.start_htd();
            sb.start_htd();
            run_pair<false>(sa, sb, rest, sigma, rsig);
            // _completion_estimate (heuristic.py:34-49) of both: CPython's sum of the
            // rest's t_k in rt order, min t_dth
            double fa = 0.0, ea = 0.0, ta = kBig, fb = 0.0, eb = 0.0, tb = kBig;
            uint64_t la = rt_drop(cand, ja), lb = rt_drop(cand, jb);
#pragma unroll 2
            for (int i = 0; i < m - 1; ++i, la >>= 4, lb >>= 4) {
                const int ua = (int)(la & 0xF), ub = (int)(lb & 0xF);
                const double xa = DV(1, ua), xb = DV(1, ub);
                const double sa_ = __dadd_rn(fa, xa), sb_ = __dadd_rn(fb, xb);
                if (sum_mode) {  // Neumaier (CPython >= 3.12): TwoSum error of f + x
                    const double pa = __dsub_rn(sa_, fa), pb = __dsub_rn(sb_, fb);
                    ea = __dadd_rn(ea, __dadd_rn(__dsub_rn(fa, __dsub_rn(sa_, pa)), __dsub_rn(xa, pa)));
                    eb = __dadd_rn(eb, __dadd_rn(__dsub_rn(fb, __dsub_rn(sb_, pb)), __dsub_rn(xb, pb)));
                }
                fa = sa_;
                fb = sb_;
                ta = dmin(DV(2, ua), ta);
                tb = dmin(DV(2, ub), tb);
            }
            if (sum_mode && ea != 0.0 && isfinite(ea)) fa = __dadd_rn(fa, ea);
            if (sum_mode && eb != 0.0 && isfinite(eb)) fb = __dadd_rn(fb, eb);
            const double bound_a = __dadd_rn(__dadd_rn(sa.kEnd, fa), ta);
            const double bound_b = __dadd_rn(__dadd_rn(sb.kEnd, fb), tb);
            const double est_a = (bound_a > sa.now) ? bound_a : sa.now;
            const double est_b = (bound_b > sb.now) ? bound_b : sb.now;
            const int ra = IR(ca), rb = IR(cb);
            if (bj < 0 || key_less(est_a, sa.idleK, ra, be, bd, br)) { bj = ja; be = est_a; bd = sa.idleK; br = ra; }
            if (two && key_less(est_b, sb.idleK, rb, be, bd, br)) { bj = jb; be = est_b; bd = sb.idleK; br = rb; }
        }
        OSIM_DCHECK(bj >= 0 && bj < m);
        const int c = rt_at(cand, bj);
        ot |= (uint64_t)c << (4 * k);
        cand = rt_drop(cand, bj);
        // advance the checkpoint by the chosen task (prefix length k + 1)
        FS s;
        s.init(base, ot, k + 1);
        s.load(ck);
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
        FS sa, sb;
        sa.init(base, ot | ((uint64_t)a << (4 * kl)) | ((uint64_t)b << (4 * (kl + 1))), n);
        sb.init(base, ot | ((uint64_t)b << (4 * kl)) | ((uint64_t)a << (4 * (kl + 1))), n);
        sa.load(ck);
        sb.load(ck);
        const int rest = __reduce_max_sync(kFull, 3 * n - sa.finalized());
        run_pair<true>(sa, sb, rest, sigma, rsig);
        const double m_ab = sa.now, m_ba = sb.now;
        bool ab;
        if (m_ab < m_ba) ab = true;
        else if (m_ba < m_ab) ab = false;
        else ab = !(DV(2, a) <= DV(2, b));  // tie: shorter DtH last
        ot |= ((uint64_t)(ab ? a : b) << (4 * kl)) | ((uint64_t)(ab ? b : a) << (4 * (kl + 1)));
        ms = ab ? m_ab : m_ba;  // simulate(ot + chosen pair)
    } else {
        FS s;  // n == 1: reorder_batch returns [tg[0]] without simulating
        s.init(base, 0, 1);
        for (int st = 0; st < 3; ++st) s.step(sigma, rsig);
        ms = s.now;
    }
    if (live) {
        ms_out[g] = ms;
        if (nsims_out) nsims_out[g] = (n >= 3) ? (uint32_t)(n * (n - 1) / 2 - 1) : (n == 2 ? 2u : 0u);
        for (int p = 0; p < n; ++p) order_out[g * (uint64_t)n + p] = (uint8_t)nib(ot, p);
    }
}

}  // namespace osim
