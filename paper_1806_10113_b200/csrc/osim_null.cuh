// osim_null.cuh -- the fast simulator generalized to null stages.
//
// A stage of duration 0 has no command (DeviceSim.submit, engine.py:129-151)
// and counts as done from the start (engine.py:133-135), so a task may skip
// its HtD, K or DtH.  NullSim keeps FastSim's register-resident state and
// op-exact arithmetic (Markstein division, sigma by multiply when a power of
// two) but:
//  * lane heads are positions (x4) of the lane's current command; after a
//    finalize the head jumps to the next position whose stage is non-null,
//    found with one find-first-set on a per-sequence null mask (bit p: the
//    stage of the task at position p is null);
//  * readiness is "head passed or stage null" (engine.py:168-178): K(p)
//    needs HtD(p) done -- p below the HtD head -- or null; DtH(p) needs the
//    same of K(p) and HtD(p); on 1-DMA the XFER queue holds the HtD slots
//    then the DtH slots (engine.py:153-154) and its DtH part starts only
//    after every HtD slot (a DtH slot is therefore always HtD-ready);
//  * the group's last command may sit in any lane, so once every lane is
//    idle dt is clamped to 0 and the remaining lock-step steps are no-ops.
// Fast-range conditions as FastSim: every non-null stage in [2^-60, 2^22)
// ms and sigma >= 2^-60, so every step finalizes at least one command.
// (NullSim itself is defined in osim_sim.cuh, next to FastSim, so the
// heuristic kernels can use it too.)
#pragma once

#include "osim_kernels.cuh"

namespace osim {

// ---------------------------------------------------------------------------
// Prefix sharing with null stages.  With nulls a suffix command can start
// before the HtD lane reaches position M (K(M) is ready at once if HtD(M) is
// null), so the checkpoint is taken in a prefix-only world (the first M
// positions): the state is prefix-determined up to the first step whose
// start phase finds some lane idle with its head at or past M -- only then
// could a position >= M command start.  Replaying a suffix restores every
// lane, rebuilds the position null masks for the full ordering, and moves
// each head that sat at M to the first non-null slot >= M of the full
// ordering (1-DMA: the prefix world's XFER slot M is the full world's HtD(M)).
// ---------------------------------------------------------------------------
template <int DMA, bool SIGP2, bool TRACK>
__device__ __forceinline__ bool null_at_ck(const NullSim<DMA, SIGP2, TRACK>& s) {
    const bool a = idle(s.r0) && s.s0 >= s.n4;  // 1-DMA prefix world: XFER at its DtH part
    const bool c = idle(s.r2) && s.s2 >= s.n4;
    if constexpr (DMA == 2) return a || c || (idle(s.r1) && s.s1 >= s.n4);
    else return a || c;
}

struct NullCk {  // structure-of-arrays checkpoint slots (conflict-free)
    double v[10][kBlock];  // now, r0, r1, r2, d0, d1, d2, c0, c1, c2
    int h[3][kBlock];      // s0, s1, s2 (prefix-world heads)
};

// Task null masks of the staged group (bit t: that stage of task t is null).
__device__ __forceinline__ void null_masks_dr(const double2* sdr, int n, unsigned& tH, unsigned& tK, unsigned& tD) {
    tH = tK = tD = 0;
    for (int t = 0; t < n; ++t) {
        tH |= (sdr[t].x > 0.0 ? 0u : 1u) << t;
        tK |= (sdr[kStride + t].x > 0.0 ? 0u : 1u) << t;
        tD |= (sdr[2 * kStride + t].x > 0.0 ? 0u : 1u) << t;
    }
}

// One prefix P (phase A in the prefix world) and its L! suffixes; leaves in
// [lo, hi) are accumulated.  Warp-collective; no block barriers.
template <int N, int DMA, bool SIGP2, int L>
__device__ __forceinline__ void null_pfx_leaves(uint32_t base, double sigma, double rsig, uint64_t P, bool validP,
                                                uint64_t lo, uint64_t hi, double thr, Part& acc,
                                                double* __restrict__ ms_out, uint64_t ms_base, NullCk& K,
                                                unsigned tH, unsigned tK, unsigned tD, int* __restrict__ err) {
    constexpr int M = N - L;
    constexpr uint64_t LF = Fact<L>::v;
    const int ti = threadIdx.x;
    const uint64_t seq0 = unrank<N>(P * LF);
    NullSim<DMA, SIGP2> s;
    // ---- phase A in the prefix-only world
    s.init(base, seq0, M, tH, tK, tD);
    int sa = 0;
#pragma unroll 1
    while (__any_sync(kFull, !null_at_ck(s) && sa < 3 * N)) {
        if (!null_at_ck(s) && sa < 3 * N) {
            s.step(sigma, rsig);
            ++sa;
        }
    }
    K.v[0][ti] = s.now; K.v[1][ti] = s.r0; K.v[2][ti] = s.r1; K.v[3][ti] = s.r2;
    K.v[4][ti] = s.d0; K.v[5][ti] = s.d1; K.v[6][ti] = s.d2;
    K.v[7][ti] = s.c0; K.v[8][ti] = s.c1; K.v[9][ti] = s.c2;
    K.h[0][ti] = s.s0; K.h[1][ti] = s.s1; K.h[2][ti] = s.s2;
    const uint64_t pre = seq0 & ((1ull << (4 * M)) - 1ull);
    const uint64_t rem = seq0 >> (4 * M);
    const int rest = 3 * N - __reduce_min_sync(kFull, validP ? sa : 3 * N);
#pragma unroll 1
    for (int j = 0; j < (int)LF; ++j) {
        uint64_t idx;
        if constexpr (L >= 4) idx = suf_tab<L>(j);
        else idx = unrank<L>((uint64_t)j);
        uint64_t suf = 0;
#pragma unroll
        for (int i = 0; i < L; ++i)
            suf |= ((rem >> (4 * ((idx >> (4 * i)) & 0xF))) & 0xFull) << (4 * (M + i));
        // ---- restore into the full world
        s.init(base, pre | suf, N, tH, tK, tD);  // full-ordering masks; state and heads below
        s.now = K.v[0][ti]; s.r0 = K.v[1][ti]; s.r1 = K.v[2][ti]; s.r2 = K.v[3][ti];
        s.d0 = K.v[4][ti]; s.d1 = K.v[5][ti]; s.d2 = K.v[6][ti];
        s.c0 = K.v[7][ti]; s.c1 = K.v[8][ti]; s.c2 = K.v[9][ti];
        const int h0 = K.h[0][ti], h1 = K.h[1][ti], h2 = K.h[2][ti];
        constexpr int M4 = 4 * M;
        using NS = NullSim<DMA, SIGP2>;
        if constexpr (DMA == 2) {
            s.s0 = h0 >= M4 ? NS::next(s.mH, M4 - 4, N) : h0;
            s.s1 = h1 >= M4 ? NS::next(s.mX, M4 - 4, N) : h1;
        } else {
            s.s0 = h0 >= M4 ? NS::next(s.mX, M4 - 4, 2 * N) : h0;
        }
        s.s2 = h2 >= M4 ? NS::next(s.mK, M4 - 4, N) : h2;
#pragma unroll 1
        for (int st = 0; st < rest; st += 2) {
            if (__all_sync(kFull, s.drained())) break;
            s.step(sigma, rsig);
            s.step(sigma, rsig);
        }
        const uint64_t r = P * LF + (uint64_t)j;
        if (validP && r >= lo && r < hi) {
            if (err && !s.drained()) atomicExch(err, OSIM_ESTALL);
            part_add<true>(acc, s.now, r, thr);
            if (ms_out) ms_out[r - ms_base] = s.now;
        }
    }
}

template <int N, int DMA, bool SIGP2, int L>
__global__ void __launch_bounds__(kBlock) k_exhaustive_null_pfx(const double* __restrict__ durs, double sigma,
                                                                uint64_t lo, uint64_t hi, double thr,
                                                                Part* __restrict__ parts,
                                                                double* __restrict__ ms_out,
                                                                int* __restrict__ err) {
    constexpr uint64_t LF = Fact<L>::v;
    __shared__ double2 sdr[3 * kStride];
    __shared__ Part sh[32];
    __shared__ NullCk K;
    stage_dr(durs, N, sdr);
    __syncthreads();
    unsigned tH, tK, tD;
    null_masks_dr(sdr, N, tH, tK, tD);
    const uint32_t base = opaque_u32((uint32_t)__cvta_generic_to_shared(sdr));  // kept in a register
    const double rsig = __ddiv_rn(1.0, sigma);
    const uint64_t p_lo = lo / LF, p_hi = (hi + LF - 1) / LF;
    Part acc;
    part_init(acc);
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t pb = p_lo + (uint64_t)blockIdx.x * blockDim.x; pb < p_hi; pb += stride) {
        const uint64_t P = pb + threadIdx.x;
        const bool validP = P < p_hi;
        null_pfx_leaves<N, DMA, SIGP2, L>(base, sigma, rsig, validP ? P : p_lo, validP, lo, hi, thr, acc, ms_out,
                                          lo, K, tH, tK, tD, err);
    }
    acc = block_reduce(acc, sh);
    if (threadIdx.x == 0) parts[blockIdx.x] = acc;
}

// Batched groups with null stages: one CTA per group.
template <int N, int DMA, bool SIGP2, int L>
__global__ void __launch_bounds__(kBlock) k_exhaustive_batch_null_pfx(const double* __restrict__ durs, uint64_t B,
                                                                      double sigma, osim_summary* __restrict__ out,
                                                                      int* __restrict__ err) {
    constexpr uint64_t total = Fact<N>::v;
    constexpr uint64_t NP = total / Fact<L>::v;
    __shared__ double2 sdr[3 * kStride];
    __shared__ Part sh[32];
    __shared__ NullCk K;
    const uint32_t base = opaque_u32((uint32_t)__cvta_generic_to_shared(sdr));  // kept in a register
    const double rsig = __ddiv_rn(1.0, sigma);
    for (uint64_t b = blockIdx.x; b < B; b += gridDim.x) {
        stage_dr(durs + b * 3 * N, N, sdr);
        __syncthreads();
        unsigned tH, tK, tD;
        null_masks_dr(sdr, N, tH, tK, tD);
        Part acc;
        part_init(acc);
        for (uint64_t pb = 0; pb < NP; pb += blockDim.x) {
            const uint64_t P = pb + threadIdx.x;
            const bool validP = P < NP;
            null_pfx_leaves<N, DMA, SIGP2, L>(base, sigma, rsig, validP ? P : 0, validP, 0, total, -kBig, acc,
                                              nullptr, 0, K, tH, tK, tD, err);
        }
        acc = block_reduce(acc, sh);  // ends with __syncthreads: smem reusable
        if (threadIdx.x == 0) out[b] = part_to_summary(acc);
    }
}

}  // namespace osim
