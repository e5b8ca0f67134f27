// osim_heur_null.cuh -- the heuristic (Algorithm 1) with prefix checkpoints
// for groups with null stages (every stage 0 or in the fast range).
//
// k_heuristic_fast's schedule (a warp owns kWG groups, a greedy round's
// candidates spread over the lanes, kLPG lanes per group for the key argmin)
// with NullSim instead of FastSim.  With null stages a command of the
// appended position can start before the HtD lane reaches it (K(k) is ready
// at once when HtD(k) is null), so a round's checkpoint is taken in the
// prefix-only world of the k chosen tasks, as the null exhaustive kernel
// does (osim_null.cuh): the state is prefix-determined up to the first step
// whose start phase finds some lane idle with its head at or past position
// k.  A candidate replay restores it into the world of k + 1 positions
// (ot + [c]) and moves every head that sat at k to the first non-null slot
// >= k of that world; the chosen task's replay, stopped at the same kind of
// point of the (k + 1)-world, is the next round's checkpoint.  Operation
// sequences per simulation are unchanged, so estimates, idle times,
// makespans and orders are bit-identical to k_heuristic<DMA, 2>.
#pragma once

#include "osim_null.cuh"

namespace osim {

struct NullHeurCk {
    double now, r0, r1, r2, d0, d1, d2, c0, c1, c2, kEnd, idleK;
    int s0, s1, s2, kfin, steps;  // prefix-world heads, K finalized yet, steps from time 0
};

template <int DMA, bool SP2>
struct NullHeurWarpShared {
    double2 dr[kWG * kHS];
    NullHeurCk ck[kWG];
    double ka[kWG * kKeyN];
    double kb[kWG * kKeyN];
    uint64_t ot[kWG];
    uint64_t cand[kWG];  // rt: remaining task ids in input order, 4 bits each
    unsigned tH[kWG], tK[kWG], tD[kWG];
    uint8_t idr[kWG * kMaxN];
};

template <class NS>
__device__ __forceinline__ void nh_save(const NS& s, int steps, NullHeurCk& k) {
    k.now = s.now; k.r0 = s.r0; k.r1 = s.r1; k.r2 = s.r2; k.d0 = s.d0; k.d1 = s.d1; k.d2 = s.d2;
    k.c0 = s.c0; k.c1 = s.c1; k.c2 = s.c2; k.kEnd = s.kEnd; k.idleK = s.idleK;
    k.s0 = s.s0; k.s1 = s.s1; k.s2 = s.s2; k.kfin = s.kfin ? 1 : 0; k.steps = steps;
}

// restore a checkpoint of the k-position prefix world into the world of the
// `len` positions of `seq` (len > k): heads that sat at k move to the first
// non-null slot >= k
template <int DMA, class NS>
__device__ __forceinline__ void nh_load(NS& s, const NullHeurCk& k, int kpos, uint32_t base, uint64_t seq, int len,
                                        unsigned tH, unsigned tK, unsigned tD) {
    s.init(base, seq, len, tH, tK, tD);
    s.now = k.now; s.r0 = k.r0; s.r1 = k.r1; s.r2 = k.r2; s.d0 = k.d0; s.d1 = k.d1; s.d2 = k.d2;
    s.c0 = k.c0; s.c1 = k.c1; s.c2 = k.c2; s.kEnd = k.kEnd; s.idleK = k.idleK; s.kfin = k.kfin != 0;
    const int M4 = 4 * kpos;
    if constexpr (DMA == 2) {
        s.s0 = k.s0 >= M4 ? NS::next(s.mH, M4 - 4, len) : k.s0;
        s.s1 = k.s1 >= M4 ? NS::next(s.mX, M4 - 4, len) : k.s1;
    } else {
        s.s0 = k.s0 >= M4 ? NS::next(s.mX, M4 - 4, 2 * len) : k.s0;
    }
    s.s2 = k.s2 >= M4 ? NS::next(s.mK, M4 - 4, len) : k.s2;
}

template <int DMA, bool SP2>
__global__ void __launch_bounds__(kHTF) k_heuristic_nullck(const double* __restrict__ durs,
                                                         const uint8_t* __restrict__ id_rank, uint64_t B, int n,
                                                         double sigma, int sum_mode, uint8_t* __restrict__ order_out,
                                                         double* __restrict__ ms_out, uint32_t* __restrict__ nsims_out,
                                                         int* __restrict__ err) {
    using SH = NullHeurWarpShared<DMA, SP2>;
    using NS = NullSim<DMA, SP2, true>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    SH& S = reinterpret_cast<SH*>(smem_raw)[warp];
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(S.dr);
    const uint64_t g0 = ((uint64_t)blockIdx.x * kWPB + warp) * kWG;
    if (g0 >= B) return;  // whole warp leaves together; no block barriers below
    const int Gv = (int)((B - g0) < (uint64_t)kWG ? (B - g0) : (uint64_t)kWG);
    const double rsig = __ddiv_rn(1.0, sigma);
    auto gbase = [&](int g) { return sbase + (uint32_t)(g * kHS * sizeof(double2)); };

    for (int i = lane; i < Gv * 3 * kStride; i += 32) {
        const int g = i / (3 * kStride), r = i % (3 * kStride);
        const int k = r / kStride, t = r % kStride;
        const double v = t < n ? durs[(g0 + g) * 3 * (uint64_t)n + 3 * t + k] : 1.0;
        S.dr[g * kHS + r] = make_double2(v, __ddiv_rn(1.0, v));
    }
    for (int i = lane; i < Gv * kMaxN; i += 32) {
        const int g = i / kMaxN, t = i % kMaxN;
        S.idr[i] = t < n ? id_rank[(g0 + g) * (uint64_t)n + t] : 0xFF;
    }
    __syncwarp();
    auto DV = [&](int g, int k, int t) { return S.dr[g * kHS + k * kStride + t].x; };
    bool ok = true;

    // select_first_task (heuristic.py:22-31), task null masks, first checkpoint
    if (lane < Gv) {
        const int g = lane;
        unsigned tH = 0, tK = 0, tD = 0;
        for (int t = 0; t < n; ++t) {
            tH |= (DV(g, 0, t) > 0.0 ? 0u : 1u) << t;
            tK |= (DV(g, 1, t) > 0.0 ? 0u : 1u) << t;
            tD |= (DV(g, 2, t) > 0.0 ? 0u : 1u) << t;
        }
        S.tH[g] = tH; S.tK[g] = tK; S.tD[g] = tD;
        const unsigned all = (1u << n) - 1u;
        unsigned rm = all;
        NS s;
        int steps = 0;
        if (n >= 3) {
            int best = -1;
            double b1 = 0, b2 = 0;
            for (int t = 0; t < n; ++t) {
                const double k1 = -__dsub_rn(DV(g, 1, t), DV(g, 0, t));
                const double k2 = -DV(g, 2, t);
                bool less;
                if (best < 0) less = true;
                else if (k1 < b1) less = true;
                else if (b1 < k1) less = false;
                else if (k2 < b2) less = true;
                else if (b2 < k2) less = false;
                else less = S.idr[g * kMaxN + t] < S.idr[g * kMaxN + best];
                if (less) { best = t; b1 = k1; b2 = k2; }
            }
            S.ot[g] = (uint64_t)best;
            rm = all & ~(1u << best);
            s.init(gbase(g), S.ot[g], 1, tH, tK, tD);  // the 1-position world
            for (; steps < 3 * kMaxN && !null_at_ck(s); ++steps) s.step(sigma, rsig);
        } else {
            S.ot[g] = 0;
            s.init(gbase(g), 0, 0, tH, tK, tD);  // the empty world: the initial state
        }
        nh_save(s, steps, S.ck[g]);
        uint64_t cl = 0;
        for (int t = n - 1; t >= 0; --t)
            if ((rm >> t) & 1u) cl = (cl << 4) | (uint64_t)t;
        S.cand[g] = cl;
    }
    __syncwarp();

    const int k0 = (n >= 3) ? 1 : 0;
    for (int k = k0; n - k > 2; ++k) {  // heuristic.py:120-123
        const int m = n - k;
        const int items = Gv * m;
        const unsigned minv = 65536u / (unsigned)m + 1u;  // i / m for i < 2^7 (see k_heuristic_fast)
        for (int i0 = 0; i0 < items; i0 += 32) {
            const int i = i0 + lane;
            const bool valid = i < items;
            const int gq = (int)(((unsigned)i * minv) >> 16);
            const int g = valid ? gq : 0;
            const int j = valid ? i - gq * m : 0;
            const uint64_t cl0 = S.cand[g];
            const int c = rt_at(cl0, j);
            NS s;
            nh_load<DMA>(s, S.ck[g], k, gbase(g), S.ot[g] | ((uint64_t)c << (4 * k)), k + 1, S.tH[g], S.tK[g],
                         S.tD[g]);
            const int rest = __reduce_max_sync(kFull, 3 * (k + 1) - S.ck[g].steps);
#pragma unroll 1
            for (int st = 0; st < rest; st += 2) {
                if (__all_sync(kFull, s.drained())) break;
                s.step(sigma, rsig);
                s.step(sigma, rsig);
            }
            ok = ok && (s.drained() || !valid);
            // _completion_estimate (heuristic.py:34-49): builtin sum of the
            // rest's t_k in rt order, min t_dth
            double f = 0.0, cmp = 0.0, tail = kBig;
            uint64_t rl = rt_drop(cl0, j);
#pragma unroll 2
            for (int q = 0; q < m - 1; ++q, rl >>= 4) {
                const int t = (int)(rl & 0xF);
                const double x = DV(g, 1, t);
                const double tt = __dadd_rn(f, x);
                if (sum_mode) {  // CPython >= 3.12: TwoSum error, as k_heuristic_fast
                    const double bp = __dsub_rn(tt, f);
                    const double e = __dadd_rn(__dsub_rn(f, __dsub_rn(tt, bp)), __dsub_rn(x, bp));
                    cmp = __dadd_rn(cmp, e);
                }
                f = tt;
                tail = dmin(DV(g, 2, t), tail);
            }
            if (sum_mode && cmp != 0.0 && isfinite(cmp)) f = __dadd_rn(f, cmp);
            const double bound = __dadd_rn(__dadd_rn(s.kEnd, f), tail);
            const double est = (bound > s.now) ? bound : s.now;
            if (valid) {
                S.ka[g * kKeyN + j] = est;
                S.kb[g * kKeyN + j] = s.idleK;
            }
        }
        __syncwarp();
        int bj;
        {
            const int g = lane / kLPG, part = lane % kLPG;
            int lj = -1;
            double le = 0, ld = 0;
            int lr = 0;
            if (g < Gv) {
                for (int j = part; j < m; j += kLPG) {
                    const double e = S.ka[g * kKeyN + j], d = S.kb[g * kKeyN + j];
                    const int r = S.idr[g * kMaxN + rt_at(S.cand[g], j)];
                    if (lj < 0 || key_less(e, d, r, le, ld, lr)) { lj = j; le = e; ld = d; lr = r; }
                }
            }
#pragma unroll
            for (int off = 1; off < kLPG; off <<= 1) {
                const int oj = __shfl_xor_sync(kFull, lj, off);
                const double oe = __shfl_xor_sync(kFull, le, off), od = __shfl_xor_sync(kFull, ld, off);
                const int orr = __shfl_xor_sync(kFull, lr, off);
                if (oj >= 0 && (lj < 0 || key_less(oe, od, orr, le, ld, lr))) { lj = oj; le = oe; ld = od; lr = orr; }
            }
            bj = __shfl_sync(kFull, lj, (lane % kWG) * kLPG);
        }
        if (lane < Gv) {  // extend the prefix, advance the checkpoint into the (k+1)-world
            const int g = lane;
            const int c = rt_at(S.cand[g], bj);
            S.ot[g] |= (uint64_t)c << (4 * k);
            S.cand[g] = rt_drop(S.cand[g], bj);
            NS s;
            nh_load<DMA>(s, S.ck[g], k, gbase(g), S.ot[g], k + 1, S.tH[g], S.tK[g], S.tD[g]);
            int steps = S.ck[g].steps;
            for (; steps < 3 * kMaxN && !null_at_ck(s); ++steps) s.step(sigma, rsig);
            nh_save(s, steps, S.ck[g]);
        }
        __syncwarp();
    }

    const int kl = n - 2;  // select_last_tasks (heuristic.py:81-102)
    double mab = 0.0;
    if (n >= 2) {
        const int i = lane;  // 2 * kWG <= 32 items
        const bool valid = i < 2 * Gv;
        const int g = valid ? i >> 1 : 0;
        const int w = i & 1;
        int a = rt_at(S.cand[g], 0), b = rt_at(S.cand[g], 1);
        if (S.idr[g * kMaxN + b] < S.idr[g * kMaxN + a]) { const int x = a; a = b; b = x; }
        const uint64_t x = w ? b : a, y = w ? a : b;
        NS s;
        nh_load<DMA>(s, S.ck[g], kl, gbase(g), S.ot[g] | (x << (4 * kl)) | (y << (4 * (kl + 1))), n, S.tH[g],
                     S.tK[g], S.tD[g]);
        const int rest = __reduce_max_sync(kFull, 3 * n - S.ck[g].steps);
#pragma unroll 1
        for (int st = 0; st < rest; st += 2) {
            if (__all_sync(kFull, s.drained())) break;
            s.step(sigma, rsig);
            s.step(sigma, rsig);
        }
        ok = ok && (s.drained() || !valid);
        if (valid) S.ka[g * kKeyN + w] = s.now;
        mab = s.now;
    }
    __syncwarp();
    (void)mab;
    if (lane < Gv) {
        const int g = lane;
        double ms;
        if (n >= 2) {
            int a = rt_at(S.cand[g], 0), b = rt_at(S.cand[g], 1);
            if (S.idr[g * kMaxN + b] < S.idr[g * kMaxN + a]) { const int x = a; a = b; b = x; }
            const double m_ab = S.ka[g * kKeyN + 0], m_ba = S.ka[g * kKeyN + 1];
            bool ab;
            if (m_ab < m_ba) ab = true;
            else if (m_ba < m_ab) ab = false;
            else ab = !(DV(g, 2, a) <= DV(g, 2, b));  // tie: shorter DtH last
            S.ot[g] |= ((uint64_t)(ab ? a : b) << (4 * kl)) | ((uint64_t)(ab ? b : a) << (4 * (kl + 1)));
            ms = ab ? m_ab : m_ba;
        } else {  // n == 1: reorder_batch returns [tg[0]] without simulating
            NS s;
            s.init(gbase(g), 0, 1, S.tH[g], S.tK[g], S.tD[g]);
            for (int st = 0; st < 3 && !s.drained(); ++st) s.step(sigma, rsig);
            ok = ok && s.drained();
            ms = s.now;
        }
        ms_out[g0 + g] = ms;
        if (nsims_out) nsims_out[g0 + g] = (n >= 3) ? (uint32_t)(n * (n - 1) / 2 - 1) : (n == 2 ? 2u : 0u);
    }
    if (!__all_sync(kFull, ok) && lane == 0) atomicExch(err, OSIM_ESTALL);
    __syncwarp();
    for (int i = lane; i < Gv * n; i += 32) {
        const int g = i / n, p = i % n;
        order_out[(g0 + g) * (uint64_t)n + p] = (uint8_t)nib(S.ot[g], p);
    }
}

}  // namespace osim
