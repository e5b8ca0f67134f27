// osim_kernels.cuh -- sm_100a kernels for the exhaustive oracle, the
// batched-group launcher and the heuristic (Algorithm 1) candidate loop.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "osim_suftab.h"
#include "osim_sim.cuh"
#include "../../include/offsim_b200.h"

namespace osim {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kBlock = 256;
#ifndef OSIM_PFX_MINB
#define OSIM_PFX_MINB 4  // min resident CTAs per SM for the prefix kernels (64 registers)
#endif

// ---------------------------------------------------------------------------
// make_report reduction (oracle.py:41-57) in mergeable form.  The product of
// makespans is carried as (mantissa in [1,2), binary exponent) instead of a
// per-ordering log: sum_log = log(lpm) + lpe*ln2 at the end.
// ---------------------------------------------------------------------------
struct Part {
    double best;
    unsigned long long rank;
    double worst;
    double sum;
    double csum;  // Neumaier compensation of sum
    double lpm;
    long long lpe;
    unsigned long long count;
    unsigned long long below;  // makespans strictly below the threshold (cli.py:102)
};

__device__ __forceinline__ void part_init(Part& a) {
    a.best = __longlong_as_double(0x7ff0000000000000ll);
    a.rank = ~0ull;
    a.worst = -__longlong_as_double(0x7ff0000000000000ll);
    a.sum = 0.0;
    a.csum = 0.0;
    a.lpm = 1.0;
    a.lpe = 0;
    a.count = 0;
    a.below = 0;
}

template <bool EXACT>
__device__ __forceinline__ void renorm(double& m, long long& e) {
    if constexpr (EXACT) {
        int ex;
        double f = frexp(m, &ex);  // f in [0.5, 1)
        m = f * 2.0;
        e += ex - 1;
    } else {
        long long bits = __double_as_longlong(m);
        e += ((bits >> 52) & 0x7ff) - 1023;
        m = __longlong_as_double((bits & 0x800FFFFFFFFFFFFFll) | (1023ll << 52));
    }
}

// compensated accumulation: s + c carries the exact running sum to ~1 ulp
// (10^8 orderings per thread block in the batch kernel at n = 12)
__device__ __forceinline__ void neumaier(double& s, double& c, double x) {
    const double t = __dadd_rn(s, x);
    c = __dadd_rn(c, (fabs(s) >= fabs(x)) ? __dadd_rn(__dsub_rn(s, t), x) : __dadd_rn(__dsub_rn(x, t), s));
    s = t;
}

// per-thread add; the lower rank wins a tie (np.argmin keeps the first of
// equal makespans), so threads may visit ranks in any order
template <bool EXACT>
__device__ __forceinline__ void part_add(Part& a, double ms, unsigned long long r, double thr) {
    if (ms < a.best || (ms == a.best && r < a.rank)) { a.best = ms; a.rank = r; }
    a.below += (ms < thr) ? 1ull : 0ull;
    a.worst = fmax(a.worst, ms);
    neumaier(a.sum, a.csum, ms);
    a.lpm = __dmul_rn(a.lpm, ms);
    renorm<EXACT>(a.lpm, a.lpe);
    a.count += 1;
}

#ifndef OSIM_LEAF_LEAN
#define OSIM_LEAF_LEAN 1
#endif
// prefix-kernel leaf: part_add without the count (added per prefix) and the
// renormalization (every 8 leaves); the threshold count only when STATS.
// LEAN (makespans are positive and finite): ranks compared in 32 bits when
// every rank fits (R32: n <= 12), the maximum without fmax's NaN handling,
// and the running sum compensated by Fast2Sum (t = s + x, error x - (t - s),
// exact whenever s >= x, i.e. from the second or third leaf of a thread on;
// the mean is not bit-exact anyway, see the reduction note in DESIGN.md)
template <bool STATS, bool R32 = false>
__device__ __forceinline__ void leaf_add(Part& a, double ms, unsigned long long r, double thr) {
#if OSIM_LEAF_LEAN
    const bool rl = R32 ? ((uint32_t)r < (uint32_t)a.rank) : (r < a.rank);
    if (ms < a.best || (ms == a.best && rl)) { a.best = ms; a.rank = r; }
    if constexpr (STATS) a.below += (ms < thr) ? 1ull : 0ull;
    a.worst = (a.worst < ms) ? ms : a.worst;
    const double t = __dadd_rn(a.sum, ms);
    a.csum = __dadd_rn(a.csum, __dsub_rn(ms, __dsub_rn(t, a.sum)));
    a.sum = t;
#else
    if (ms < a.best || (ms == a.best && r < a.rank)) { a.best = ms; a.rank = r; }
    if constexpr (STATS) a.below += (ms < thr) ? 1ull : 0ull;
    a.worst = fmax(a.worst, ms);
    neumaier(a.sum, a.csum, ms);
#endif
    a.lpm = __dmul_rn(a.lpm, ms);
}

// order-independent for best/rank (lexicographic), fixed tree order for sums
__device__ __forceinline__ void part_merge(Part& a, const Part& b) {
    if (b.best < a.best || (b.best == a.best && b.rank < a.rank)) { a.best = b.best; a.rank = b.rank; }
    a.worst = fmax(a.worst, b.worst);
    neumaier(a.sum, a.csum, b.sum);
    a.csum = __dadd_rn(a.csum, b.csum);
    a.lpm = __dmul_rn(a.lpm, b.lpm);
    a.lpe += b.lpe;
    renorm<false>(a.lpm, a.lpe);
    a.count += b.count;
    a.below += b.below;
}

__device__ __forceinline__ Part part_shfl(const Part& a, int m) {
    Part b;
    b.best = __shfl_xor_sync(kFull, a.best, m);
    b.rank = __shfl_xor_sync(kFull, a.rank, m);
    b.worst = __shfl_xor_sync(kFull, a.worst, m);
    b.sum = __shfl_xor_sync(kFull, a.sum, m);
    b.csum = __shfl_xor_sync(kFull, a.csum, m);
    b.lpm = __shfl_xor_sync(kFull, a.lpm, m);
    b.lpe = __shfl_xor_sync(kFull, a.lpe, m);
    b.count = __shfl_xor_sync(kFull, a.count, m);
    b.below = __shfl_xor_sync(kFull, a.below, m);
    return b;
}

// Block reduce (all threads call; blockDim.x multiple of 32); result valid
// in thread 0.  Deterministic: xor-tree in the warp, then warps in order.
__device__ __forceinline__ Part block_reduce(Part a, Part* sh /*[32]*/) {
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) {
        Part b = part_shfl(a, m);
        // keep the tree symmetric: lower lane merges the higher lane's value
        if ((threadIdx.x & m) == 0) part_merge(a, b);
        else { Part c = b; part_merge(c, a); a = c; }
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) sh[w] = a;
    __syncthreads();
    if (w == 0) {
        const int nw = blockDim.x >> 5;
        if (l < nw) a = sh[l]; else part_init(a);
#pragma unroll
        for (int m = 16; m >= 1; m >>= 1) {
            Part b = part_shfl(a, m);
            if ((threadIdx.x & m) == 0) part_merge(a, b);
            else { Part c = b; part_merge(c, a); a = c; }
        }
    }
    __syncthreads();
    return a;
}

__device__ __forceinline__ osim_summary part_to_summary(const Part& a) {
    osim_summary s;
    s.best = a.best;
    s.best_rank = a.rank;
    s.worst = a.worst;
    s.sum = __dadd_rn(a.sum, a.csum);
    s.sum_log = a.count ? log(a.lpm) + (double)a.lpe * 0.6931471805599453094 : 0.0;
    s.count = a.count;
    return s;
}

// Stage one group's durations into kind-major shared rows + reciprocals.
__device__ __forceinline__ void stage_durs(const double* __restrict__ g, int n, double* sd, double* sr) {
    for (int i = threadIdx.x; i < 3 * kStride; i += blockDim.x) {
        const int k = i / kStride, t = i % kStride;
        const double v = t < n ? g[3 * t + k] : 1.0;
        sd[i] = v;
        sr[i] = __ddiv_rn(1.0, v);  // RN(1/v): the Markstein reciprocal
    }
}

__device__ __forceinline__ void null_masks(const double* sd, int n, unsigned& nH, unsigned& nK,
                                           unsigned& nD) {
    nH = nK = nD = 0;
    for (int t = 0; t < n; ++t) {
        if (!(sd[0 * kStride + t] > 0.0)) nH |= 1u << t;
        if (!(sd[1 * kStride + t] > 0.0)) nK |= 1u << t;
        if (!(sd[2 * kStride + t] > 0.0)) nD |= 1u << t;
    }
}

// Warp-uniform run loop: the warp steps until all its lanes drained.
template <class S>
__device__ __forceinline__ void run_warp(S& s, int max_steps) {
#pragma unroll 1
    for (int st = 0; st < max_steps; ++st) {
        if (__all_sync(kFull, s.drained())) break;
        s.step();
    }
}

// ---------------------------------------------------------------------------
// Exhaustive search, general path (null stages or out-of-range durations):
// one thread per ordering, Lehmer-unranked, IEEE division.
// ---------------------------------------------------------------------------
template <int DMA>
__global__ void __launch_bounds__(kBlock) k_exhaustive_gen(const double* __restrict__ durs, int n,
                                                           double sigma, uint64_t lo, uint64_t hi, double thr,
                                                           Part* __restrict__ parts,
                                                           double* __restrict__ ms_out,
                                                           int* __restrict__ err) {
    __shared__ double sd[3 * kStride], sr[3 * kStride];
    __shared__ Part sh[32];
    stage_durs(durs, n, sd, sr);
    __syncthreads();
    unsigned nH, nK, nD;
    null_masks(sd, n, nH, nK, nD);
    const Durs D{sd, sr};
    Part acc;
    part_init(acc);
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t base = lo + (uint64_t)blockIdx.x * blockDim.x; base < hi; base += stride) {
        const uint64_t r = base + threadIdx.x;
        const bool valid = r < hi;
        Sim<DMA, false, false, false> s;
        s.init(D, unrank_rt(valid ? r : lo, n), n, sigma, 1.0, nH, nK, nD);
        run_warp(s, 3 * n * kSlowSteps);
        if (!s.drained()) atomicExch(err, OSIM_ESTALL);
        if (valid) {
            part_add<true>(acc, s.now, r, thr);
            if (ms_out) ms_out[r - lo] = s.now;
        }
    }
    acc = block_reduce(acc, sh);
    if (threadIdx.x == 0) parts[blockIdx.x] = acc;
}

// Deterministic final reduce of per-block partials (fixed order).
static __global__ void __launch_bounds__(kBlock) k_final_reduce(const Part* __restrict__ parts, int P,
                                                         osim_summary* __restrict__ out,
                                                         unsigned long long* __restrict__ below) {
    __shared__ Part sh[32];
    Part a;
    part_init(a);
    for (int i = threadIdx.x; i < P; i += blockDim.x) part_merge(a, parts[i]);
    a = block_reduce(a, sh);
    if (threadIdx.x == 0) {
        *out = part_to_summary(a);
        if (below) *below = a.below;
    }
}

// ---------------------------------------------------------------------------
// Prefix-sharing exhaustive search (fast path).
// Lexicographic rank order groups orderings by prefix: ranks
// [P*L!, (P+1)*L!) share positions 0..M-1 (M = N-L) and permute the L
// remaining tasks.  Everything the simulator does before the HtD (XFER) lane
// is free to start position M depends only on positions 0..M-1: a command
// of position >= M can only start after HtD(M) started, and HtD(M) starts
// the step after HtD(M-1) finalized (both FIFOs hold the ordering in
// position order; on a 1-DMA device every DtH queues behind every HtD).  So
// a thread simulates its prefix once up to that checkpoint (phase A), keeps
// the register state, and replays only the L! suffixes from it (phase B).
// The per-ordering operation sequence is unchanged, so results are
// bit-identical to simulating each ordering from time 0.
// ---------------------------------------------------------------------------
template <int L>
struct Fact {
    static constexpr uint64_t v = (uint64_t)L * Fact<L - 1>::v;
};
template <>
struct Fact<0> {
    static constexpr uint64_t v = 1;
};

__device__ __forceinline__ void stage_dr(const double* __restrict__ g, int n, double2* sdr) {
    for (int i = threadIdx.x; i < 3 * kStride; i += blockDim.x) {
        const int k = i / kStride, t = i % kStride;
        const double v = t < n ? g[3 * t + k] : 1.0;
        sdr[i] = make_double2(v, __ddiv_rn(1.0, v));
    }
}

#ifdef OSIM_HSTATS
// lane-slot counters of lock-step replays (tools/heur_lanes.py, tools/pfx_lanes.py):
// 32 x warp replay length, steps each lane needs, the same for the full-step
// phase, empty-lane slots, replays, sum of warp replay lengths and full phases
__device__ unsigned long long g_hstats[8];
template <class FS>
__device__ __forceinline__ void hstats_replay(const FS& s, int rest, bool valid, double sigma, double rsig) {
    FS t = s;
    int h1 = 0, own = 0;
    for (int q = 0; q < rest; ++q) {
        if (t.s0 < t.n4) ++h1;
        if (!t.drained()) ++own;
        t.step(sigma, rsig);
    }
    const int mh1 = __reduce_max_sync(kFull, h1);
    const unsigned vb = __ballot_sync(kFull, valid);
    const int sown = __reduce_add_sync(kFull, valid ? own : 0);
    const int sh1 = __reduce_add_sync(kFull, valid ? h1 : 0);
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&g_hstats[0], (unsigned long long)(32 * rest));
        atomicAdd(&g_hstats[1], (unsigned long long)sown);
        atomicAdd(&g_hstats[2], (unsigned long long)(32 * mh1));
        atomicAdd(&g_hstats[3], (unsigned long long)sh1);
        atomicAdd(&g_hstats[4], (unsigned long long)((32 - __popc(vb)) * rest));
        atomicAdd(&g_hstats[5], 1ull);
        atomicAdd(&g_hstats[6], (unsigned long long)rest);
        atomicAdd(&g_hstats[7], (unsigned long long)mh1);
    }
}
#endif

// Per-thread checkpoint slots in shared memory, structure-of-arrays so that
// the 32 lanes of a warp touch 32 consecutive 8-byte words (conflict-free);
// keeping them out of registers lifts occupancy.  At a checkpoint the HtD lane
// has just finalized (rem = sentinel, head known to the caller), so only the
// DtH and K lanes and the clock are stored: 7 doubles + 2 ints per thread.
template <int SLOTS>
struct CkSlots {
    double v[SLOTS][7][kBlock];  // now, r1, r2, d1, d2, c1, c2
    int h[SLOTS][2][kBlock];     // s1, s2
};

template <int SLOTS, class FS>
__device__ __forceinline__ void ck_store(CkSlots<SLOTS>& K, int slot, int i, const FS& s) {
    K.v[slot][0][i] = s.now; K.v[slot][1][i] = s.r1; K.v[slot][2][i] = s.r2;
    K.v[slot][3][i] = s.d1; K.v[slot][4][i] = s.d2; K.v[slot][5][i] = s.c1; K.v[slot][6][i] = s.c2;
    K.h[slot][0][i] = s.s1; K.h[slot][1][i] = s.s2;
}
// restore; the HtD lane is idle with `hdone` HtDs finalized
template <int SLOTS, class FS>
__device__ __forceinline__ void ck_load(const CkSlots<SLOTS>& K, int slot, int i, FS& s, int hdone) {
    s.now = K.v[slot][0][i]; s.r1 = K.v[slot][1][i]; s.r2 = K.v[slot][2][i];
    s.d1 = K.v[slot][3][i]; s.d2 = K.v[slot][4][i]; s.c1 = K.v[slot][5][i]; s.c2 = K.v[slot][6][i];
    s.s1 = K.h[slot][0][i]; s.s2 = K.h[slot][1][i];
    s.r0 = kBig;
    s.s0 = 4 * hdone;
}

constexpr int kPfxQ = 2;  // prefixes per thread and prefix-kernel call
#ifndef OSIM_SUBCK
#define OSIM_SUBCK 1
#endif
#ifndef OSIM_SUB_MINN
#define OSIM_SUB_MINN 11  // sub-checkpoints for groups of at least this many tasks
#endif
#ifndef OSIM_SUB_D1
#define OSIM_SUB_D1 0     // ... and on 1-DMA devices
#endif
#ifndef OSIM_SUB_SNAP
#define OSIM_SUB_SNAP 1   // the sub-checkpoint is stored by the group's first leaf (no separate advance)
#endif
// Checkpoint slots of the prefix kernels, two kinds.  Full (CkSlots): the
// clock, the K/DtH rems and their {nd, 1/nd} (7 doubles + 2 ints per slot).
// Compact (PfxCkC, 2-DMA when OSIM_SUBCK): only the clock, the rems and the
// heads (3 doubles + 2 ints); the running commands' {nd, 1/nd} are reloaded
// from the duration rows by their task (the K/DtH heads), which needs the
// sequence set first -- and one more slot per thread holds the
// sub-checkpoint one HtD later (see pfx_leaves).  Both fit the same dynamic
// shared memory (kPfxCkBytes).
struct PfxCkC {
    double v[kPfxQ + 1][3][kBlock];  // now, r1, r2; slot kPfxQ: the sub-checkpoint
    int h[kPfxQ + 1][2][kBlock];     // s1, s2
};
template <class T> struct CkNV { static constexpr int v = 7; };
template <> struct CkNV<PfxCkC> { static constexpr int v = 3; };
template <bool C> struct PfxCkSel { using T = CkSlots<kPfxQ>; };
template <> struct PfxCkSel<true> { using T = PfxCkC; };
constexpr size_t kPfxCkBytes =
    sizeof(PfxCkC) > sizeof(CkSlots<kPfxQ>) ? sizeof(PfxCkC) : sizeof(CkSlots<kPfxQ>);
template <class FS>
__device__ __forceinline__ void pk_store(PfxCkC& K, int slot, int i, const FS& s) {
    K.v[slot][0][i] = s.now; K.v[slot][1][i] = s.r1; K.v[slot][2][i] = s.r2;
    K.h[slot][0][i] = s.s1; K.h[slot][1][i] = s.s2;
}
// restore (s.seq set): the HtD lane idle with `hdone` HtDs finalized
template <class FS>
__device__ __forceinline__ void pk_load(const PfxCkC& K, int slot, int i, FS& s, int hdone) {
    s.now = K.v[slot][0][i]; s.r1 = K.v[slot][1][i]; s.r2 = K.v[slot][2][i];
    s.s1 = K.h[slot][0][i]; s.s2 = K.h[slot][1][i];
    s.r0 = kBig;
    s.s0 = 4 * hdone;
    s.reload_kd();
}
template <class FS>
__device__ __forceinline__ void pk_store(CkSlots<kPfxQ>& K, int slot, int i, const FS& s) { ck_store(K, slot, i, s); }
template <class FS>
__device__ __forceinline__ void pk_load(const CkSlots<kPfxQ>& K, int slot, int i, FS& s, int hdone) {
    ck_load(K, slot, i, s, hdone);
}

// Advance every lane of the warp to the checkpoint "htd_done() == target";
// returns this lane's step count.
template <class FS>
__device__ __forceinline__ int advance_to(FS& s, int target, double sigma, double rsig) {
    int n = 0;
#pragma unroll 1
    // (<= 3n steps on fast-eligible data; the bound keeps ineligible input finite)
    while (__any_sync(kFull, s.htd_done() < target && n < 3 * kMaxN)) {
        if (s.htd_done() < target && n < 3 * kMaxN) {
            s.step(sigma, rsig);
            ++n;
        }
    }
    return n;
}

// Phase-B lanes of a warp run in lock-step for 3N - min(sa) steps, sa being
// a lane's phase-A step count, so lanes with a larger sa idle through no-op
// steps.  Each call therefore takes kPfxQ = 2 prefixes per thread (512 per
// CTA), sorts the 512 checkpoints by sa (a deterministic counting sort:
// per-warp bins from __match_any_sync, ties by entry index) and cuts the
// sorted list into 16 chunks of 32; warp w replays chunk w and chunk 15 - w,
// so lanes of a chunk have nearly equal remaining length (C4: executed /
// needed replay steps 1.095 -> ~1.01) while every warp gets a similar total
// (one long and one short chunk), which keeps the CTA's barrier waits short.
// Entries without a prefix (range tails) sort last; all-empty chunks are
// skipped.
// a value the compiler cannot rematerialize inside the replay loops (it keeps
// the register instead of recomputing the shared-window base every iteration)
__device__ __forceinline__ uint32_t opaque_u32(uint32_t x) {
#ifndef OSIM_NO_OPAQUE
    uint32_t y;
    asm volatile("mov.b32 %0, %1;" : "=r"(y) : "r"(x));
    return y;
#else
    return x;
#endif
}

#ifndef OSIM_SJT
#define OSIM_SJT 1
#endif
#ifndef OSIM_SJT_PIN
#define OSIM_SJT_PIN 1
#endif
// swap the nibbles at suffix positions p and p + 1 of a packed sequence whose
// suffix position 0 starts at bit SH0 (p warp-uniform); when the L suffix
// nibbles lie in the high word (N = 12 with the pre-shift: bits 36..51) the
// swap is 32-bit: two shifts, a masked xor, a multiply and an xor
template <int SH0, int L>
__device__ __forceinline__ void swap_nibbles(uint64_t& v, int p) {
    const int sh = SH0 + 4 * p;
    if constexpr (SH0 >= 32 && SH0 + 4 * L <= 64) {
        uint32_t h = (uint32_t)(v >> 32);
        const int s = sh - 32;
        const uint32_t x = ((h >> s) ^ (h >> (s + 4))) & 0xFu;
        h ^= x * (0x11u << s);
        v = (v & 0xFFFFFFFFull) | ((uint64_t)h << 32);
    } else {
        const uint64_t x = ((v >> sh) ^ (v >> (sh + 4))) & 0xFull;
        v ^= (x * 0x11ull) << sh;
    }
}

constexpr int kSaBins = 64;  // sa <= 3 * kMaxN; bin kSaBins - 1 = no prefix
// FastSim LAYOUT of the prefix kernels' duration rows: 0 (address = register
// base + kind offset + task offset) or 4 (base | task offset, one LOP3); both
// with the base in a register the compiler cannot rematerialize (opaque_u32).
// Measured (tools/exh_ab.py): C4 20.80 G (0) vs 20.62 G (4); C2 22.20 G (0) vs
// 22.86 G (4); with the base rematerialized each iteration (round 1) 20.35 / 22.50.
#ifndef OSIM_PFX_LAYOUT
#define OSIM_PFX_LAYOUT 0  // k_exhaustive_pfx
#endif
#ifndef OSIM_BATCH_LAYOUT
#define OSIM_BATCH_LAYOUT 4  // k_exhaustive_batch_pfx
#endif
constexpr int kNW = kBlock / 32;
struct PfxSort {
    uint64_t seq[kPfxQ * kBlock];
    uint64_t P[kPfxQ * kBlock];  // ~0: no prefix
    int sa[kPfxQ * kBlock];
    int cnt[kPfxQ][kNW][kSaBins];
    int base[kSaBins];
    short order[kPfxQ * kBlock];
};

// Sort this CTA's kPfxQ * 256 entries (entry e = q * 256 + thread) by sa;
// returns the entries this thread replays (chunks w and 2 * kNW - 1 - w).
__device__ __forceinline__ int2 pfx_sort(PfxSort& S, int sa0, int sa1) {
    const int ti = threadIdx.x, lane = ti & 31, w = ti >> 5;
    for (int i = lane; i < kSaBins; i += 32) {
        S.cnt[0][w][i] = 0;
        S.cnt[1][w][i] = 0;
    }
    __syncwarp();
    const unsigned m0 = __match_any_sync(kFull, sa0), m1 = __match_any_sync(kFull, sa1);
    if (lane == __ffs(m0) - 1) S.cnt[0][w][sa0] = __popc(m0);
    if (lane == __ffs(m1) - 1) S.cnt[1][w][sa1] = __popc(m1);
    __syncthreads();
    if (w == 0) {
        int carry = 0;
#pragma unroll
        for (int b0 = 0; b0 < kSaBins; b0 += 32) {
            const int b = b0 + lane;
            int t = 0;
#pragma unroll
            for (int q = 0; q < kPfxQ; ++q)
#pragma unroll
                for (int ww = 0; ww < kNW; ++ww) t += S.cnt[q][ww][b];
            int x = t;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(kFull, x, o);
                if (lane >= o) x += y;
            }
            S.base[b] = carry + x - t;
            carry += __shfl_sync(kFull, x, 31);
        }
    }
    __syncthreads();
    const unsigned lt = (1u << lane) - 1u;
    int r0 = S.base[sa0] + __popc(m0 & lt);
    int r1 = S.base[sa1] + __popc(m1 & lt);
    for (int ww = 0; ww < kNW; ++ww) {
        if (ww < w) r0 += S.cnt[0][ww][sa0];
        r1 += S.cnt[0][ww][sa1] + (ww < w ? S.cnt[1][ww][sa1] : 0);
    }
    OSIM_DCHECK(sa0 >= 0 && sa0 < kSaBins && sa1 >= 0 && sa1 < kSaBins);
    OSIM_DCHECK(r0 >= 0 && r0 < kPfxQ * kBlock && r1 >= 0 && r1 < kPfxQ * kBlock && r0 != r1);
    S.order[r0] = (short)ti;
    S.order[r1] = (short)(kBlock + ti);
    __syncthreads();
    const int2 e = make_int2(S.order[32 * w + lane], S.order[32 * (2 * kNW - 1 - w) + lane]);
    OSIM_DCHECK(e.x >= 0 && e.x < kPfxQ * kBlock && e.y >= 0 && e.y < kPfxQ * kBlock);
    return e;
}

// Simulate this CTA's prefixes P0 + t and P0 + 256 + t (t = thread) of
// length M and every suffix; accumulate leaves that fall inside [lo, hi) and
// below prefix p_end.  All threads of the CTA must call together.
// (A further checkpoint level two positions later was measured slower on B200:
// its middle segment runs in divergent advance loops shared by only two
// leaves.)
template <int N, int DMA, bool SIGP2, int L, bool STATS, int LAY>
__device__ __forceinline__ void pfx_leaves(uint32_t base, double sigma, double rsig, uint64_t P0, uint64_t p_end,
                                           uint64_t lo, uint64_t hi, double thr, Part& acc,
                                           double* __restrict__ ms_out, uint64_t ms_base, unsigned char* dsm,
                                           PfxSort& S) {
    constexpr int M = N - L;
    constexpr bool kC = OSIM_SUBCK && (DMA == 2 || OSIM_SUB_D1);  // compact slots (+ sub-checkpoints)
    // steps per phase vote in the full phase: 3 measured best for the
    // cheaper power-of-two-sigma step at n >= 10 (C4 +0.9 %), 2 otherwise
    // (sigma 0.375: 3 is -1.5 %; C2, n = 8: -0.4 %)
    constexpr int kPhF = (SIGP2 && N >= 10) ? OSIM_PH_FULL_P2 : OSIM_PH_FULL;
    using CK = typename PfxCkSel<kC>::T;
    constexpr int kCkV = CkNV<CK>::v;
    CK& K = *reinterpret_cast<CK*>(dsm);
    constexpr uint64_t LF = Fact<L>::v;
    using FS = FastSim<DMA, SIGP2, false, (N <= 15), false, LAY>;
    const int ti = threadIdx.x;
    FS s;
    // ---- phase A: both prefixes to their checkpoints
    int sa[kPfxQ];
#pragma unroll
    for (int q = 0; q < kPfxQ; ++q) {
        const uint64_t P = P0 + (uint64_t)q * kBlock + ti;
        const bool valid = P < p_end;
        const uint64_t seq0 = unrank<N>((valid ? P : P0) * LF);  // prefix + ascending remainder
        s.init(base, seq0, N);
        int a = 0;
        if constexpr (M > 0) {
            a = advance_to(s, valid ? M : 0, sigma, rsig);
            pk_store(K, q, ti, s);
        }
        OSIM_DCHECK(a >= 0 && a < kSaBins - 1);
        sa[q] = valid ? a : kSaBins - 1;
        S.seq[q * kBlock + ti] = seq0;
        S.P[q * kBlock + ti] = valid ? P : ~0ull;
        S.sa[q * kBlock + ti] = sa[q];
    }
    // ---- reassign: this thread replays entries e.x then e.y
    const int2 e = pfx_sort(S, sa[0], sa[1]);
    uint64_t seqq[kPfxQ], Pq[kPfxQ];
    double tu[kCkV], tv[kCkV];
    int tg[2], th[2];
    {
        const int ex = e.x & (kBlock - 1), qx = e.x >> 8;
        const int ey = e.y & (kBlock - 1), qy = e.y >> 8;
        static_assert(kBlock == 256, "entry index split");
        seqq[0] = S.seq[e.x]; Pq[0] = S.P[e.x]; sa[0] = S.sa[e.x];
        seqq[1] = S.seq[e.y]; Pq[1] = S.P[e.y]; sa[1] = S.sa[e.y];
        if constexpr (kC && M > 0) {  // raw copies (a compact restore needs the sequence)
#pragma unroll
            for (int k = 0; k < kCkV; ++k) { tu[k] = K.v[qx][k][ex]; tv[k] = K.v[qy][k][ey]; }
            tg[0] = K.h[qx][0][ex]; tg[1] = K.h[qx][1][ex];
            th[0] = K.h[qy][0][ey]; th[1] = K.h[qy][1][ey];
            __syncthreads();  // every source slot has been read
#pragma unroll
            for (int k = 0; k < kCkV; ++k) { K.v[0][k][ti] = tu[k]; K.v[1][k][ti] = tv[k]; }
            K.h[0][0][ti] = tg[0]; K.h[0][1][ti] = tg[1];
            K.h[1][0][ti] = th[0]; K.h[1][1][ti] = th[1];
        } else if constexpr (M > 0) {
            (void)tu; (void)tg;
            ck_load(K, qx, ex, s, M);
#pragma unroll
            for (int k = 0; k < kCkV; ++k) tv[k] = K.v[qy][k][ey];
            th[0] = K.h[qy][0][ey];
            th[1] = K.h[qy][1][ey];
            __syncthreads();  // every source slot has been read
            ck_store(K, 0, ti, s);
#pragma unroll
            for (int k = 0; k < kCkV; ++k) K.v[1][k][ti] = tv[k];
            K.h[1][0][ti] = th[0];
            K.h[1][1][ti] = th[1];
        } else {
            (void)tu; (void)tg; (void)tv; (void)th;
            __syncthreads();
        }
    }
    // ---- phase B: replay the L! suffixes of each taken prefix
#pragma unroll 1
    for (int q = 0; q < kPfxQ; ++q) {
        const bool validP = Pq[q] != ~0ull;
        if (!__any_sync(kFull, validP)) continue;  // all-empty chunk (range tail)
        const uint64_t P = validP ? Pq[q] : 0ull;
        const uint64_t seq0 = seqq[q];
        const uint64_t pre = (M > 0) ? (seq0 & ((1ull << (4 * M)) - 1ull)) : 0ull;
        const uint64_t rem = seq0 >> (4 * M);  // L ascending task ids
        const int rest = 3 * N - __reduce_min_sync(kFull, validP ? sa[q] : 3 * N);
        // leaves [r0, r0 + L!) of this prefix that fall inside [lo, hi)
        const uint64_t r0 = P * LF;
        const bool any_in = validP && r0 + LF > lo && r0 < hi;
        const bool all_in = validP && r0 >= lo && r0 + LF <= hi;
        if (any_in) acc.count += (r0 + LF < hi ? r0 + LF : hi) - (r0 > lo ? r0 : lo);
        // sub-checkpoints: the (L-1)! leaves that share the first suffix task
        // f also share the replay up to f's HtD finalize, so it runs once per
        // f -- the group's first leaf stores the state in the thread's sub
        // slot as it passes it (OSIM_SUB_SNAP; else a lock-step advance) --
        // and the other leaves replay only from there; the L-1 later tasks in
        // adjacent-swap order, ranks f * (L-1)! + the table's
        if constexpr (kC && L >= 3 && M > 0 && N >= OSIM_SUB_MINN) {
            constexpr int L1 = L - 1;
            constexpr uint64_t LF1 = Fact<L1>::v;
            constexpr int kSh1 = 4 * (M + 1) + (FS::kPre ? 4 : 0);  // bit of suffix position 1
#pragma unroll 1
            for (int f = 0; f < L; ++f) {
                const uint64_t lowm = (1ull << (4 * f)) - 1ull;
                const uint64_t others = (rem & lowm) | ((rem >> (4 * (f + 1))) << (4 * f));  // ascending
                const uint64_t suf = ((rem >> (4 * f)) & 0xFull) | (others << 4);
                uint64_t cur = FS::pack_seq(pre | (suf << (4 * M)));
#if OSIM_SUB_SNAP
                // the group's first leaf replays from the prefix checkpoint and
                // leaves the sub-checkpoint behind as it passes it
                int af = 0;
                int restf = rest;
#else
                s.seq = cur;
                pk_load(K, q, ti, s, M);
                const int af = advance_to(s, validP ? M + 1 : 0, sigma, rsig);
                pk_store(K, kPfxQ, ti, s);
                const int restf = 3 * N - __reduce_min_sync(kFull, validP ? sa[q] + af : 3 * N);
#endif
#pragma unroll 1
                for (int j = 0; j < (int)LF1; ++j) {
                    const uint32_t tj = sjt_tab<L1>(j);
                    const int lj = f * (int)LF1 + (int)(tj & 0xFFu);  // lexicographic leaf index
                    const uint64_t r = r0 + (uint64_t)(OSIM_SJT_PIN ? opaque_u32((uint32_t)lj) : (uint32_t)lj);
                    s.seq = cur;
#if OSIM_SUB_SNAP
                    if (j == 0) {
                        pk_load(K, q, ti, s, M);
                        swap_nibbles<kSh1, L1>(cur, (int)(tj >> 8));
                        s.template run_phased_snap<kPhF>(rest, sigma, rsig, M + 1, [&](int stp) {
                            pk_store(K, kPfxQ, ti, s);
                            af = stp;
                        });
                    } else {
                        if (j == 1) restf = 3 * N - __reduce_min_sync(kFull, validP ? sa[q] + af : 3 * N);
                        pk_load(K, kPfxQ, ti, s, M + 1);
                        swap_nibbles<kSh1, L1>(cur, (int)(tj >> 8));
                        s.template run_phased<true, kPhF>(restf, sigma, rsig);
                    }
#else
                    pk_load(K, kPfxQ, ti, s, M + 1);
                    swap_nibbles<kSh1, L1>(cur, (int)(tj >> 8));
                    s.template run_phased<true, kPhF>(restf, sigma, rsig);
#endif
                    if (all_in || (any_in && r >= lo && r < hi)) {
                        leaf_add<STATS, (N <= 12)>(acc, s.now, r, thr);
                        if constexpr (STATS) {
                            OSIM_DCHECK(r >= ms_base && r >= lo && r < hi);
                            if (ms_out) ms_out[r - ms_base] = s.now;
                        }
                    }
                    const int k = f * (int)LF1 + j;  // leaves done in this prefix, minus one
                    if ((k & 7) == 7 || k == (int)LF - 1) renorm<false>(acc.lpm, acc.lpe);
                }
            }
            continue;
        }
#if OSIM_SJT
        // the L! suffixes in adjacent-swap (Steinhaus-Johnson-Trotter) order:
        // each leaf's sequence is the previous one with two neighbouring
        // nibbles swapped (sjt_tab: the leaf's lexicographic rank and the swap
        // to the next), instead of composing L nibbles from a rank
        uint64_t cur = FS::pack_seq(pre | (rem << (4 * M)));  // the identity suffix, rank 0
        constexpr int kSh0 = 4 * M + (FS::kPre ? 4 : 0);     // bit of suffix position 0 in cur
#endif
#pragma unroll 1
        for (int j = 0; j < (int)LF; ++j) {
#if OSIM_SJT
            // (the rank is taken here, ahead of the replay, instead of
            // the table load being sunk to its first use after it; pinning the
            // whole entry instead moved the swap off the uniform datapath)
            const uint32_t tj = sjt_tab<L>(j);
            const uint32_t rj = OSIM_SJT_PIN ? opaque_u32(tj & 0xFFu) : (tj & 0xFFu);
            const uint64_t r = r0 + (uint64_t)rj;  // (the swap below keeps tj uniform)
            if constexpr (M > 0) {
                s.seq = cur;
                pk_load(K, q, ti, s, M);
            } else {
                s.init(base, 0, N);
                s.seq = cur;
            }
            swap_nibbles<kSh0, L>(cur, (int)(tj >> 8));  // the next leaf's sequence
#else
            // suffix order: for L >= 4 a constant-table load replaces ~35
            // uniform-datapath instructions per leaf (+1 % at N = 12); for
            // short suffixes the inline unrank measured faster (the load's
            // latency sits on the shorter replays' critical path)
            uint64_t idx;
            if constexpr (L >= 4) idx = suf_tab<L>(j);
            else idx = unrank<L>((uint64_t)j);
            uint64_t suf = 0;
#pragma unroll
            for (int i = 0; i < L; ++i) {
                const uint32_t id = (uint32_t)(idx >> (4 * i)) & 0xFu;
                suf |= ((rem >> (4 * id)) & 0xFull) << (4 * (M + i));
            }
            s.set_seq(pre | suf);
            if constexpr (M > 0) pk_load(K, q, ti, s, M);
            else s.init(base, 0, N), s.set_seq(pre | suf);
            const uint64_t r = r0 + (uint64_t)j;
#endif
            // full steps while any lane of the warp still has an HtD to run, then
            // K+DtH steps, then DtH-only steps (FastSim::run_phased)
#ifdef OSIM_HSTATS
            hstats_replay(s, rest, validP, sigma, rsig);
#endif
            s.template run_phased<true, kPhF>(rest, sigma, rsig);
            if (all_in || (any_in && r >= lo && r < hi)) {
                leaf_add<STATS, (N <= 12)>(acc, s.now, r, thr);
                if constexpr (STATS) {
                    OSIM_DCHECK(r >= ms_base && r >= lo && r < hi);
                    if (ms_out) ms_out[r - ms_base] = s.now;
                }
            }
            // the log-product's exponent is split off every 8 leaves (exact:
            // only the binary exponent moves; a fast-path makespan lies in
            // [2^-60, 2^88] -- durations in [2^-60, 2^22), sigma >= 2^-60,
            // n <= 16 -- so 8 of them times the mantissa in [1, 2) stay within
            // [2^-480, 2^705], inside the normal range)
            if ((j & 7) == 7 || j == (int)LF - 1) renorm<false>(acc.lpm, acc.lpe);
        }
    }
    // No trailing barrier: after the copy above every K slot is read only by
    // its owner, and the shared arrays pfx_sort reads across threads are
    // rewritten in the next call only after that call's first barrier -- a
    // warp done early runs its next phase A meanwhile.
}

// The last CTA to finish reduces every CTA's partial (the work of
// k_final_reduce, same thread mapping and tree, so the same bits) and resets
// the counter: one launch per search instead of two.  `done` must be 0 on
// entry; `parts` are read past L1 (written by other CTAs).
__device__ __forceinline__ void fused_final_reduce(const Part* parts, osim_summary* out, unsigned long long* below,
                                                   unsigned* done, Part* sh) {
    __shared__ bool last;
    __syncthreads();  // this CTA's partial is written (thread 0 wrote it)
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned prev = atomicAdd(done, 1u);
        OSIM_DCHECK(prev < gridDim.x);  // the counter starts at 0 and is reset by the last CTA
        last = prev == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    Part a;
    part_init(a);
    for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) {
        const volatile Part& p = parts[i];
        Part b;
        b.best = p.best; b.rank = p.rank; b.worst = p.worst; b.sum = p.sum; b.csum = p.csum;
        b.lpm = p.lpm; b.lpe = p.lpe; b.count = p.count; b.below = p.below;
        part_merge(a, b);
    }
    a = block_reduce(a, sh);
    if (threadIdx.x == 0) {
        *out = part_to_summary(a);
        if (below) *below = a.below;
        *done = 0u;
    }
}

// dynamic shared memory of the prefix kernels (checkpoint slots + sort)
constexpr size_t kPfxDynSmem = kPfxCkBytes + sizeof(PfxSort);

template <int N, int DMA, bool SIGP2, int L, bool STATS>
__global__ void __launch_bounds__(kBlock, OSIM_PFX_MINB) k_exhaustive_pfx(const double* __restrict__ durs, double sigma,
                                                           uint64_t lo, uint64_t hi, double thr, Part* __restrict__ parts,
                                                           double* __restrict__ ms_out, osim_summary* __restrict__ out,
                                                           unsigned long long* __restrict__ below,
                                                           unsigned* __restrict__ done, unsigned shard,
                                                           unsigned shards, unsigned split) {
    __shared__ __align__(256) double2 sdr[3 * kStride];  // 256-aligned: FastSim LAYOUT 4
    __shared__ Part sh[32];
    extern __shared__ __align__(16) unsigned char pfx_dsm[];
    PfxSort& S = *reinterpret_cast<PfxSort*>(pfx_dsm + kPfxCkBytes);
    stage_dr(durs, N, sdr);
    __syncthreads();
    const uint32_t base = opaque_u32((uint32_t)__cvta_generic_to_shared(sdr));
    const double rsig = __ddiv_rn(1.0, sigma);
    constexpr uint64_t LF = Fact<L>::v;
    const uint64_t p_lo = lo / LF, p_hi = (hi + LF - 1) / LF;
    Part acc;
    part_init(acc);
    constexpr uint64_t kPer = (uint64_t)kPfxQ * kBlock;  // prefixes per CTA call
    // grid-stride over calls of 512 prefixes.  (An even split of the ragged
    // last round over all CTAs measured slower: a CTA left alone on an SM by
    // the partial wave runs ~3x faster than one sharing it, so the grid-stride
    // tail costs only a fraction of a call.)  Interleaved shards (shards > 1,
    // osim_exhaustive_shard_dev): this launch takes calls shard, shard +
    // shards, ... of the range, so every shard samples the whole rank space
    // and the per-shard work evens out.
    // split = 2 (small shards): CTAs 2c and 2c + 1 share call c, 256
    // prefixes each (the second prefix slot of every thread stays empty and
    // sorts last), so the partition into calls is the same for any split.
    const uint64_t per = kPer / split;
    const uint64_t cta_call = blockIdx.x / split, half = blockIdx.x % split;
    const uint64_t stride = (uint64_t)(gridDim.x / split) * kPer * shards;
    for (uint64_t pc = p_lo + (cta_call * shards + shard) * kPer; pc < p_hi; pc += stride) {
        const uint64_t pb = pc + half * per;
        const uint64_t pe = pb + per < p_hi ? pb + per : p_hi;
        if (pb < pe) pfx_leaves<N, DMA, SIGP2, L, STATS, OSIM_PFX_LAYOUT>(base, sigma, rsig, pb, pe, lo, hi, thr, acc, ms_out, lo, pfx_dsm, S);
    }
    acc = block_reduce(acc, sh);
    if (threadIdx.x == 0) parts[blockIdx.x] = acc;
    if (out) fused_final_reduce(parts, out, below, done, sh);
}

// Batched groups with prefix sharing: one CTA per group.
template <int N, int DMA, bool SIGP2, int L>
__global__ void __launch_bounds__(kBlock, OSIM_PFX_MINB) k_exhaustive_batch_pfx(const double* __restrict__ durs, uint64_t B,
                                                                 double sigma, osim_summary* __restrict__ out) {
    __shared__ __align__(256) double2 sdr[3 * kStride];  // 256-aligned: FastSim LAYOUT 4
    __shared__ Part sh[32];
    extern __shared__ __align__(16) unsigned char pfx_dsm[];
    PfxSort& S = *reinterpret_cast<PfxSort*>(pfx_dsm + kPfxCkBytes);
    constexpr uint64_t total = Fact<N>::v;
    constexpr uint64_t NP = total / Fact<L>::v;
    constexpr uint64_t kPer = (uint64_t)kPfxQ * kBlock;
    const uint32_t base = opaque_u32((uint32_t)__cvta_generic_to_shared(sdr));
    const double rsig = __ddiv_rn(1.0, sigma);
    for (uint64_t b = blockIdx.x; b < B; b += gridDim.x) {
        stage_dr(durs + b * 3 * N, N, sdr);
        __syncthreads();
        Part acc;
        part_init(acc);
        for (uint64_t pb = 0; pb < NP; pb += kPer)
            pfx_leaves<N, DMA, SIGP2, L, false, OSIM_BATCH_LAYOUT>(base, sigma, rsig, pb, NP, 0, total, -kBig, acc, nullptr, 0, pfx_dsm, S);
        acc = block_reduce(acc, sh);  // ends with __syncthreads: smem reusable
        if (threadIdx.x == 0) out[b] = part_to_summary(acc);
    }
}

// ---------------------------------------------------------------------------
// Explicit orderings (sampled mode, oracle.py:127-135): thread per ordering.
// ---------------------------------------------------------------------------
template <int DMA, bool FAST>
__global__ void __launch_bounds__(kBlock) k_eval_perms(const double* __restrict__ durs, int n,
                                                       double sigma,
                                                       const uint8_t* __restrict__ perms,
                                                       uint64_t cnt, double thr, double* __restrict__ ms_out,
                                                       Part* __restrict__ parts,
                                                       int* __restrict__ err) {
    __shared__ double sd[3 * kStride], sr[3 * kStride];
    __shared__ Part sh[32];
    stage_durs(durs, n, sd, sr);
    __syncthreads();
    unsigned nH = 0, nK = 0, nD = 0;
    if constexpr (!FAST) null_masks(sd, n, nH, nK, nD);
    const double rsig = __ddiv_rn(1.0, sigma);
    const Durs D{sd, sr};
    Part acc;
    part_init(acc);
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < cnt; base += stride) {
        const uint64_t i = base + threadIdx.x;
        const bool valid = i < cnt;
        const uint8_t* p = perms + (valid ? i : 0) * (uint64_t)n;
        uint64_t seq = 0;
        for (int j = 0; j < n; ++j) seq |= (uint64_t)(p[j] & 0xF) << (4 * j);
        Sim<DMA, FAST, FAST, false> s;
        s.init(D, seq, n, sigma, rsig, nH, nK, nD);
        run_warp(s, 3 * n * kSlowSteps);
        if (!s.drained()) atomicExch(err, OSIM_ESTALL);
        if (valid) {
            part_add<!FAST>(acc, s.now, i, thr);
            ms_out[i] = s.now;
        }
    }
    acc = block_reduce(acc, sh);
    if (threadIdx.x == 0) parts[blockIdx.x] = acc;
}

// Batched groups, general path: one CTA per group, n! orderings per CTA.
template <int DMA>
__global__ void __launch_bounds__(kBlock) k_exhaustive_batch_gen(const double* __restrict__ durs,
                                                                 uint64_t B, int n, double sigma,
                                                                 osim_summary* __restrict__ out,
                                                                 int* __restrict__ err) {
    __shared__ double sd[3 * kStride], sr[3 * kStride];
    __shared__ Part sh[32];
    uint64_t total = 1;
    for (int i = 2; i <= n; ++i) total *= (uint64_t)i;
    for (uint64_t b = blockIdx.x; b < B; b += gridDim.x) {
        stage_durs(durs + b * 3 * (uint64_t)n, n, sd, sr);
        __syncthreads();
        unsigned nH, nK, nD;
        null_masks(sd, n, nH, nK, nD);
        const Durs D{sd, sr};
        Part acc;
        part_init(acc);
        for (uint64_t base = 0; base < total; base += blockDim.x) {
            const uint64_t r = base + threadIdx.x;
            const bool valid = r < total;
            Sim<DMA, false, false, false> s;
            s.init(D, unrank_rt(valid ? r : 0, n), n, sigma, 1.0, nH, nK, nD);
            run_warp(s, 3 * n * kSlowSteps);
            if (!s.drained()) atomicExch(err, OSIM_ESTALL);
            if (valid) part_add<true>(acc, s.now, r, -kBig);
        }
        acc = block_reduce(acc, sh);
        if (threadIdx.x == 0) out[b] = part_to_summary(acc);
    }
}

// ---------------------------------------------------------------------------
// One ordering with its full timeline (engine.simulate, engine.py:252-263).
// ---------------------------------------------------------------------------
template <int DMA>
__global__ void k_timeline(const double* __restrict__ durs, int n, double sigma,
                           const uint8_t* __restrict__ order, double* start, double* end,
                           double* res /*[4] makespan, idle HtD, K, DtH*/, int* err) {
    __shared__ double sd[3 * kStride], sr[3 * kStride];
    stage_durs(durs, n, sd, sr);
    __syncthreads();
    if (threadIdx.x != 0) return;
    unsigned nH, nK, nD;
    null_masks(sd, n, nH, nK, nD);
    for (int i = 0; i < 3 * n; ++i) { start[i] = -1.0; end[i] = -1.0; }
    uint64_t seq = 0;
    for (int j = 0; j < n; ++j) seq |= (uint64_t)(order[j] & 0xF) << (4 * j);
    Sim<DMA, false, false, false> s;
    s.init(Durs{sd, sr}, seq, n, sigma, 1.0, nH, nK, nD);
    TimelineOut tl{start, end};
    if (!s.run(&tl)) { *err = OSIM_ESTALL; return; }
    res[0] = s.now;
    // idle_report (engine.py:68-80): each kind's spans in FIFO order, which
    // is their (start, end) order
    for (int k = 0; k < 3; ++k) {
        double idle = 0.0, prev_end = 0.0;
        bool any = false;
        for (int j = 0; j < n; ++j) {
            const int t = order[j];
            if (start[3 * t + k] < 0.0) continue;
            const double st = start[3 * t + k];
            if (any && st > prev_end) idle = __dadd_rn(idle, __dsub_rn(st, prev_end));
            prev_end = end[3 * t + k];
            any = true;
        }
        res[1 + k] = idle;
    }
}

// ---------------------------------------------------------------------------
// Heuristic (Algorithm 1, heuristic.py:105-125) for many groups.
// CTA-cooperative: a CTA owns G groups in shared memory; every greedy round
// all groups have the same prefix length k, so the round's G*(n-k)
// candidate simulations (select_next_task, heuristic.py:71-77) have equal
// length and are spread over all threads in lock-step; one thread per
// group then takes the argmin of (estimate, idle_K, id) and extends the
// prefix.
// ---------------------------------------------------------------------------
constexpr int kHG = 32;     // groups per CTA
constexpr int kHT = 128;    // threads per CTA
constexpr int kHS = 49;     // double2 per group: [3][16] {nd, 1/nd} + 1 pad (bank spread)

struct HeurShared {
    double2 dr[kHG * kHS];
    double ka[kHG * kMaxN];
    double kb[kHG * kMaxN];
    uint64_t ot[kHG];
    unsigned rmask[kHG];
    unsigned nH[kHG], nK[kHG], nD[kHG];
    uint8_t idr[kHG * kMaxN];
    uint8_t cand[kHG * kMaxN];
    uint8_t pa[kHG], pb[kHG];
};

// One simulation of `seq` (len positions) of group g from time 0.  MODE 1:
// FastSim (no null stage); MODE 2: NullSim (null stages, fast range); MODE 0:
// the general simulator (IEEE division, any durations).
template <int DMA, int MODE, bool TRACK>
struct HeurRun {
    double ms, kEnd, idleK;
    bool ok;
    __device__ __forceinline__ void run(HeurShared& S, uint32_t sbase, int g, uint64_t seq, int len, double sigma,
                                        double rsig, bool sp2) {
        if constexpr (MODE == 1) {
            const uint32_t base = sbase + (uint32_t)(g * kHS * sizeof(double2));
            if (sp2 && DMA == 2) {
                FastSim<DMA, true, TRACK, false> s;
                s.init(base, seq, len);
#pragma unroll 1
                for (int st = 0; st < 3 * len; ++st) s.step(sigma, rsig);
                ms = s.now; kEnd = s.kEnd; idleK = s.idleK; ok = s.drained();
            } else {
                FastSim<DMA, false, TRACK, false> s;
                s.init(base, seq, len);
#pragma unroll 1
                for (int st = 0; st < 3 * len; ++st) s.step(sigma, rsig);
                ms = s.now; kEnd = s.kEnd; idleK = s.idleK; ok = s.drained();
            }
        } else if constexpr (MODE == 2) {
            const uint32_t base = sbase + (uint32_t)(g * kHS * sizeof(double2));
            if (sp2 && DMA == 2) {
                NullSim<DMA, true, TRACK> s;
                s.init(base, seq, len, S.nH[g], S.nK[g], S.nD[g]);
#pragma unroll 1
                for (int st = 0; st < 3 * len; ++st) s.step(sigma, rsig);
                ms = s.now; kEnd = s.kEnd; idleK = s.idleK; ok = s.drained();
            } else {
                NullSim<DMA, false, TRACK> s;
                s.init(base, seq, len, S.nH[g], S.nK[g], S.nD[g]);
#pragma unroll 1
                for (int st = 0; st < 3 * len; ++st) s.step(sigma, rsig);
                ms = s.now; kEnd = s.kEnd; idleK = s.idleK; ok = s.drained();
            }
        } else {
            const double* p = reinterpret_cast<const double*>(&S.dr[g * kHS]);
            Sim<DMA, false, false, TRACK> s;
            s.init(Durs{p, p + 1, 2}, seq, len, sigma, rsig, S.nH[g], S.nK[g], S.nD[g]);
            run_warp(s, 3 * len * kSlowSteps);
            ms = s.now; kEnd = s.kEnd; idleK = s.idleK; ok = s.drained();
        }
    }
};

template <int DMA, int MODE>
__global__ void __launch_bounds__(kHT) k_heuristic(const double* __restrict__ durs,
                                                   const uint8_t* __restrict__ id_rank, uint64_t B,
                                                   int n, double sigma, int sum_mode,
                                                   uint8_t* __restrict__ order_out,
                                                   double* __restrict__ ms_out,
                                                   uint32_t* __restrict__ nsims_out,
                                                   int* __restrict__ err) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    HeurShared& S = *reinterpret_cast<HeurShared*>(smem_raw);
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(S.dr);
    const uint64_t g0 = (uint64_t)blockIdx.x * kHG;
    const int Gv = (int)((B - g0) < (uint64_t)kHG ? (B - g0) : (uint64_t)kHG);
    const double rsig = __ddiv_rn(1.0, sigma);
    int se;
    const bool sp2 = frexp(sigma, &se) == 0.5;
    const int tid = threadIdx.x;

    // stage durations ({nd, 1/nd}, kind-major rows) + id ranks
    for (int i = tid; i < Gv * 3 * kStride; i += blockDim.x) {
        const int g = i / (3 * kStride), r = i % (3 * kStride);
        const int k = r / kStride, t = r % kStride;
        const double v = t < n ? durs[(g0 + g) * 3 * (uint64_t)n + 3 * t + k] : 1.0;
        S.dr[g * kHS + r] = make_double2(v, __ddiv_rn(1.0, v));
    }
    for (int i = tid; i < Gv * kMaxN; i += blockDim.x) {
        const int g = i / kMaxN, t = i % kMaxN;
        S.idr[i] = t < n ? id_rank[(g0 + g) * (uint64_t)n + t] : 0xFF;
    }
    __syncthreads();

    auto DV = [&](int g, int k, int t) { return S.dr[g * kHS + k * kStride + t].x; };

    // select_first_task (heuristic.py:22-31): min over rt of
    // (-(t_k - t_htd), -t_dth, id)
    if (tid < Gv) {
        const int g = tid;
        unsigned nH = 0, nK = 0, nD = 0;
        for (int t = 0; t < n; ++t) {
            if (!(DV(g, 0, t) > 0.0)) nH |= 1u << t;
            if (!(DV(g, 1, t) > 0.0)) nK |= 1u << t;
            if (!(DV(g, 2, t) > 0.0)) nD |= 1u << t;
        }
        S.nH[g] = nH; S.nK[g] = nK; S.nD[g] = nD;
        unsigned all = (n >= 32) ? ~0u : ((1u << n) - 1u);
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
            S.rmask[g] = all & ~(1u << best);
        } else {
            S.ot[g] = 0;
            S.rmask[g] = all;
        }
        int c = 0;
        for (int t = 0; t < n; ++t)
            if ((S.rmask[g] >> t) & 1u) S.cand[g * kMaxN + c++] = (uint8_t)t;
    }
    __syncthreads();

    const int k0 = (n >= 3) ? 1 : 0;  // prefix length after the first pick
    // greedy rounds: while len(rt) > 2 (heuristic.py:120-123)
    for (int k = k0; n - k > 2; ++k) {
        const int m = n - k;
        const int items = Gv * m;
        for (int i0 = 0; i0 < items; i0 += blockDim.x) {
            const int i = i0 + tid;
            const bool valid = i < items;
            const int g = valid ? i / m : 0;
            const int j = valid ? i % m : 0;
            const int c = S.cand[g * kMaxN + j];
            const uint64_t seq = S.ot[g] | ((uint64_t)c << (4 * k));
            HeurRun<DMA, MODE, true> hr;
            hr.run(S, sbase, g, seq, k + 1, sigma, rsig, sp2);
            // _completion_estimate (heuristic.py:34-49); rest in rt order
            PySum ps;
            ps.reset();
            double tail = 0.0;
            bool any = false;
            const unsigned rest = S.rmask[g] & ~(1u << c);
            for (int t = 0; t < n; ++t) {
                if (!((rest >> t) & 1u)) continue;
                ps.add(DV(g, 1, t), sum_mode);
                const double d = DV(g, 2, t);
                if (!any || d < tail) tail = d;
                any = true;
            }
            const double bound = __dadd_rn(__dadd_rn(hr.kEnd, ps.result(sum_mode)), tail);
            const double est = (bound > hr.ms) ? bound : hr.ms;
            if (valid) {
                S.ka[g * kMaxN + j] = est;
                S.kb[g * kMaxN + j] = hr.idleK;
            }
        }
        __syncthreads();
        if (tid < Gv) {
            const int g = tid;
            int bj = 0;
            for (int j = 1; j < m; ++j) {
                const double e = S.ka[g * kMaxN + j], be = S.ka[g * kMaxN + bj];
                const double d = S.kb[g * kMaxN + j], bd = S.kb[g * kMaxN + bj];
                bool less;
                if (e < be) less = true;
                else if (be < e) less = false;
                else if (d < bd) less = true;
                else if (bd < d) less = false;
                else less = S.idr[g * kMaxN + S.cand[g * kMaxN + j]] <
                            S.idr[g * kMaxN + S.cand[g * kMaxN + bj]];
                if (less) bj = j;
            }
            const int c = S.cand[g * kMaxN + bj];
            S.ot[g] |= (uint64_t)c << (4 * k);
            S.rmask[g] &= ~(1u << c);
            int cc = 0;
            for (int t = 0; t < n; ++t)
                if ((S.rmask[g] >> t) & 1u) S.cand[g * kMaxN + cc++] = (uint8_t)t;
        }
        __syncthreads();
    }

    const int kl = n - 2;  // select_last_tasks (heuristic.py:81-102)
    if (n >= 2) {
        if (tid < Gv) {
            const int g = tid;
            int a = S.cand[g * kMaxN + 0], b = S.cand[g * kMaxN + 1];
            if (S.idr[g * kMaxN + b] < S.idr[g * kMaxN + a]) { int x = a; a = b; b = x; }
            S.pa[g] = (uint8_t)a;
            S.pb[g] = (uint8_t)b;
        }
        __syncthreads();
        for (int i0 = 0; i0 < 2 * Gv; i0 += blockDim.x) {
            const int i = i0 + tid;
            const bool valid = i < 2 * Gv;
            const int g = valid ? i >> 1 : 0;
            const int w = i & 1;
            const uint64_t x = w ? S.pb[g] : S.pa[g], y = w ? S.pa[g] : S.pb[g];
            const uint64_t seq = S.ot[g] | (x << (4 * kl)) | (y << (4 * (kl + 1)));
            HeurRun<DMA, MODE, false> hr;
            hr.run(S, sbase, g, seq, n, sigma, rsig, sp2);
            if (valid) S.ka[g * kMaxN + w] = hr.ms;
        }
        __syncthreads();
        if (tid < Gv) {
            const int g = tid;
            const int a = S.pa[g], b = S.pb[g];
            const double m_ab = S.ka[g * kMaxN + 0], m_ba = S.ka[g * kMaxN + 1];
            bool ab;
            if (m_ab < m_ba) ab = true;
            else if (m_ba < m_ab) ab = false;
            else ab = !(DV(g, 2, a) <= DV(g, 2, b));  // tie: shorter DtH last
            S.ot[g] |= ((uint64_t)(ab ? a : b) << (4 * kl)) | ((uint64_t)(ab ? b : a) << (4 * (kl + 1)));
        }
        __syncthreads();
    }

    // final ordering, its makespan and the simulation count
    for (int i0 = 0; i0 < Gv; i0 += blockDim.x) {
        const int i = i0 + tid;
        const bool valid = i < Gv;
        const int g = valid ? i : 0;
        HeurRun<DMA, MODE, false> hr;
        hr.run(S, sbase, g, S.ot[g], n, sigma, rsig, sp2);
        if (!hr.ok) atomicExch(err, OSIM_ESTALL);
        if (valid) {
            ms_out[g0 + g] = hr.ms;
            if (nsims_out) nsims_out[g0 + g] = (n >= 3) ? (uint32_t)(n * (n - 1) / 2 - 1) : (n == 2 ? 2u : 0u);
        }
    }
    for (int i = tid; i < Gv * n; i += blockDim.x) {
        const int g = i / n, p = i % n;
        order_out[(g0 + g) * (uint64_t)n + p] = (uint8_t)nib(S.ot[g], p);
    }
}

// ---------------------------------------------------------------------------
// Heuristic, all-stages-non-null path with prefix checkpoints.
// Same CTA-cooperative schedule as k_heuristic, plus: every candidate
// simulation of a greedy round is `simulate(ot + [cand])`, and the state of
// that simulation up to the step in which the HtD lane frees up after
// position len(ot)-1 depends on `ot` only (the argument of
// k_exhaustive_pfx).  Each group keeps that state in shared memory; the
// round's candidates start from it, and after the argmin one thread per
// group advances it by the chosen task.  The final pair's two simulations
// start from the last checkpoint and their makespans are the reported
// makespan of the chosen ordering.  Per-simulation operation sequences are
// unchanged, so every estimate, idle time and makespan is bit-identical.
// ---------------------------------------------------------------------------
#ifndef OSIM_HWG
#define OSIM_HWG 8
#endif
// candidate keys: per-lane registers (lane owns group lane % kWG; 7 CTAs/SM)
// unless -DOSIM_HKSHARED (keys in shared memory, group-major items; 6 CTAs/SM)
#if !defined(OSIM_HKSHARED) && !defined(OSIM_HKREG)
#define OSIM_HKREG 1
#endif
constexpr int kWG = OSIM_HWG;          // groups per warp
constexpr int kLPG = 32 / kWG;         // lanes per group in the key argmin
constexpr int kKeyN = kMaxN - 1;       // candidates per greedy round (n - k, k >= 1)
constexpr int kWPB = 32 / kWG;         // warps per CTA
constexpr int kHGF = kWG * kWPB;       // groups per CTA (fast kernel)
constexpr int kHTF = 32 * kWPB;        // threads per CTA (fast kernel)
static_assert(kLPG * kWG == 32 && kWG <= 16, "groups per warp");

#ifndef OSIM_HSPLIT
#define OSIM_HSPLIT 1  // k_heuristic_fast, 2-DMA: command starts as three 8-byte loads (start_if_split;
                       // C5 NVIDIA 147.4 -> 150.4, AMD 143.1 -> 147.9 M decisions/s; PHI 172.3 -> 168.6)
#endif
template <int DMA, bool SP2>
struct HeurWarpShared {
    using FS = FastSim<DMA, SP2, true, false, false, (OSIM_HSPLIT != 0 && DMA == 2) ? 1 : 0>;  // 1-DMA: measured slower
    double2 dr[kWG * kHS];
    typename FS::Ck ck[kWG];
#ifndef OSIM_HKREG
    double ka[kWG * kKeyN];  // per-candidate keys (m <= 15 per round)
    double kb[kWG * kKeyN];
#else
    double ka[kWG * 2];  // the final pair's makespans only
#endif
    uint64_t ot[kWG];
    uint64_t cand[kWG];  // rt: remaining task ids in input order, 4 bits each
    uint8_t idr[kWG * kMaxN];
    uint8_t pa[kWG], pb[kWG];
};

// packed rt list: entry j, and the list without entry j (order kept)
__device__ __forceinline__ int rt_at(uint64_t l, int j) { return (int)((l >> (4 * j)) & 0xF); }
__device__ __forceinline__ uint64_t rt_drop(uint64_t l, int j) {
    return (l & ((1ull << (4 * j)) - 1ull)) | ((l >> (4 * j + 4)) << (4 * j));
}

// (estimate, idle_K, id rank) key of select_next_task (heuristic.py:74-76)
__device__ __forceinline__ bool key_less(double e, double d, int r, double be, double bd, int br) {
    if (e < be) return true;
    if (be < e) return false;
    if (d < bd) return true;
    if (bd < d) return false;
    return r < br;
}

#ifndef OSIM_HMINB
#define OSIM_HMINB 0  // min resident CTAs per SM for k_heuristic_fast (0: unspecified; register budget, tuning)
#endif
#if OSIM_HMINB > 0
#define OSIM_HLB __launch_bounds__(kHTF, OSIM_HMINB)
#else
#define OSIM_HLB __launch_bounds__(kHTF)
#endif
template <int DMA, bool SP2>
__global__ void OSIM_HLB k_heuristic_fast(const double* __restrict__ durs,
                                                        const uint8_t* __restrict__ id_rank, uint64_t B, int n,
                                                        double sigma, int sum_mode,
                                                        uint8_t* __restrict__ order_out,
                                                        double* __restrict__ ms_out,
                                                        uint32_t* __restrict__ nsims_out) {
    using SH = HeurWarpShared<DMA, SP2>;
    using FS = typename SH::FS;
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
#ifndef OSIM_HKREG
    constexpr int KA = kKeyN;
#else
    constexpr int KA = 2;
#endif

    // select_first_task (heuristic.py:22-31) and the first checkpoint
    if (lane < Gv) {
        const int g = lane;
        const unsigned all = (1u << n) - 1u;
        unsigned rm;
        FS s;
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
            s.init(gbase(g), S.ot[g], 1);
            for (int q = 0; q < 3 * kMaxN && s.htd_done() < 1; ++q) s.step(sigma, rsig);
        } else {
            S.ot[g] = 0;
            rm = all;
            s.init(gbase(g), 0, 1);  // empty prefix: the initial state
        }
        s.save(S.ck[g]);
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
        // i / m for i < 2^7 by a 16-bit reciprocal: (i * (2^16/m + 1)) >> 16
        // is exact (the excess i/2^16 < 2^-9 stays below 1/m)
#ifndef OSIM_HKREG
        const unsigned minv = 65536u / (unsigned)m + 1u;
        for (int i0 = 0; i0 < items; i0 += 32) {
            const int i = i0 + lane;
            const bool valid = i < items;
            const int gq = (int)(((unsigned)i * minv) >> 16);
            const int g = valid ? gq : 0;
            const int j = valid ? i - gq * m : 0;
#else
        // lane owns group lane % kWG and candidates j = lane / kWG + kLPG * it;
        // its best key is kept in registers across the iterations
        (void)items;
        int lj = -1;
        double le = 0, ld = 0;
        int lr = 0;
        for (int j0 = 0; j0 < m; j0 += kLPG) {
            const int jq = j0 + lane / kWG;
            const bool valid = (lane % kWG) < Gv && jq < m;
            const int g = valid ? lane % kWG : 0;
            const int j = valid ? jq : 0;
#endif
            const uint64_t cl0 = S.cand[g];
            const int c = rt_at(cl0, j);
            OSIM_DCHECK(g >= 0 && g < kWG && j >= 0 && j < m && c >= 0 && c < n);
            OSIM_DCHECK(!valid || ((S.ot[g] >> (4 * k)) == 0ull));  // position k is still free
            FS s;
            s.init(gbase(g), S.ot[g] | ((uint64_t)c << (4 * k)), k + 1);
            s.load(S.ck[g]);
            const int rest = __reduce_max_sync(kFull, 3 * (k + 1) - s.finalized());
#ifdef OSIM_HSTATS
            hstats_replay(s, rest, valid, sigma, rsig);
#endif
            s.start_htd();  // the candidate's HtD, the only one left
            s.template run_phased<false>(rest, sigma, rsig);
            // _completion_estimate (heuristic.py:34-49): builtin sum of the
            // rest's t_k in rt order (cand[] is rt in input order, rest skips
            // position j), min t_dth.  Warp-uniform loop over the m-1 rest.
            double f = 0.0, cmp = 0.0, tail = kBig;
            uint64_t rl = rt_drop(cl0, j);
#pragma unroll 2
            for (int i = 0; i < m - 1; ++i, rl >>= 4) {
                const int t = (int)(rl & 0xF);
                const double2 kd = make_double2(DV(g, 1, t), DV(g, 2, t));
                const double x = kd.x;
                const double tt = __dadd_rn(f, x);
                if (sum_mode) {  // Neumaier (CPython >= 3.12); f = 0 first is 0 + x0
                    // CPython adds the exact rounding error of f + x, computed
                    // by Fast2Sum on the (larger, smaller) magnitude pair;
                    // TwoSum yields the same exact error without the select
                    const double bp = __dsub_rn(tt, f);
                    const double e = __dadd_rn(__dsub_rn(f, __dsub_rn(tt, bp)), __dsub_rn(x, bp));
                    cmp = __dadd_rn(cmp, e);
                }
                f = tt;
                tail = dmin(kd.y, tail);
            }
            if (sum_mode && cmp != 0.0 && isfinite(cmp)) f = __dadd_rn(f, cmp);
            const double bound = __dadd_rn(__dadd_rn(s.kEnd, f), tail);
            const double est = (bound > s.now) ? bound : s.now;
#ifndef OSIM_HKREG
            if (valid) {
                S.ka[g * kKeyN + j] = est;
                S.kb[g * kKeyN + j] = s.idleK;
            }
#else
            if (valid) {
                const int r = S.idr[g * kMaxN + c];
                if (lj < 0 || key_less(est, s.idleK, r, le, ld, lr)) { lj = j; le = est; ld = s.idleK; lr = r; }
            }
#endif
        }
        __syncwarp();
        // argmin of the key over the m candidates (a strict total order, so the
        // reduction order is immaterial).  Register path (default): each lane
        // already holds the best key of its candidates j = lane / kWG + kLPG *
        // it of group lane % kWG; shuffles across the lanes with the same
        // lane % kWG leave group g's argmin on lane g.
        int bj;
#ifdef OSIM_HKREG
        {
#pragma unroll
            for (int off = kWG; off < 32; off <<= 1) {
                const int oj = __shfl_xor_sync(kFull, lj, off);
                const double oe = __shfl_xor_sync(kFull, le, off), od = __shfl_xor_sync(kFull, ld, off);
                const int orr = __shfl_xor_sync(kFull, lr, off);
                if (oj >= 0 && (lj < 0 || key_less(oe, od, orr, le, ld, lr))) { lj = oj; le = oe; ld = od; lr = orr; }
            }
            bj = lj;  // lane < kWG holds group `lane`'s argmin
        }
#else
        // shared-key path (-DOSIM_HKSHARED): kLPG lanes per group, each
        // scanning every kLPG-th candidate's key in shared memory, then a
        // shuffle reduction over the group's kLPG lanes
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
            bj = __shfl_sync(kFull, lj, (lane % kWG) * kLPG);  // group `lane` (< kWG) result
        }
#endif
        if (lane < Gv) {
            const int g = lane;
            const int c = rt_at(S.cand[g], bj);
            S.ot[g] |= (uint64_t)c << (4 * k);
            OSIM_DCHECK(bj >= 0 && bj < m);
            S.cand[g] = rt_drop(S.cand[g], bj);
            // advance the checkpoint by the chosen task (prefix length k+1)
            FS s;
            s.init(gbase(g), S.ot[g], k + 1);
            s.load(S.ck[g]);
            // bounded: the optimistic host pass may run this on ineligible input
            s.start_htd();  // the chosen task's HtD, the queue's last
            if constexpr (DMA == 2) {
                for (int q = 0; q < 3 * kMaxN && s.htd_done() < k + 1; ++q) s.template step<false>(sigma, rsig);
            } else {
                for (int q = 0; q < 3 * kMaxN && s.htd_done() < k + 1; ++q) s.step_1dk();
            }
            s.save(S.ck[g]);
        }
        __syncwarp();
    }

    const int kl = n - 2;  // select_last_tasks (heuristic.py:81-102)
    if (n >= 2) {
        if (lane < Gv) {
            const int g = lane;
            int a = rt_at(S.cand[g], 0), b = rt_at(S.cand[g], 1);
            if (S.idr[g * kMaxN + b] < S.idr[g * kMaxN + a]) { int x = a; a = b; b = x; }
            S.pa[g] = (uint8_t)a;
            S.pb[g] = (uint8_t)b;
        }
        __syncwarp();
        {
            const int i = lane;  // 2 * kWG <= 32 items
            const bool valid = i < 2 * Gv;
            const int g = valid ? i >> 1 : 0;
            const int w = i & 1;
            const uint64_t x = w ? S.pb[g] : S.pa[g], y = w ? S.pa[g] : S.pb[g];
            FS s;
            s.init(gbase(g), S.ot[g] | (x << (4 * kl)) | (y << (4 * (kl + 1))), n);
            s.load(S.ck[g]);
            const int rest = __reduce_max_sync(kFull, 3 * n - s.finalized());
            s.run_phased(rest, sigma, rsig);
            if (valid) S.ka[g * KA + w] = s.now;
        }
        __syncwarp();
    }
    if (lane < Gv) {
        const int g = lane;
        double ms;
        if (n >= 2) {
            const int a = S.pa[g], b = S.pb[g];
            const double m_ab = S.ka[g * KA + 0], m_ba = S.ka[g * KA + 1];
            bool ab;
            if (m_ab < m_ba) ab = true;
            else if (m_ba < m_ab) ab = false;
            else ab = !(DV(g, 2, a) <= DV(g, 2, b));  // tie: shorter DtH last
            S.ot[g] |= ((uint64_t)(ab ? a : b) << (4 * kl)) | ((uint64_t)(ab ? b : a) << (4 * (kl + 1)));
            ms = ab ? m_ab : m_ba;  // simulate(ot + chosen pair)
        } else {
            FS s;  // n == 1: reorder_batch returns [tg[0]] without simulating
            s.init(gbase(g), 0, 1);
            for (int st = 0; st < 3; ++st) s.step(sigma, rsig);
            ms = s.now;
        }
        ms_out[g0 + g] = ms;
        if (nsims_out) nsims_out[g0 + g] = (n >= 3) ? (uint32_t)(n * (n - 1) / 2 - 1) : (n == 2 ? 2u : 0u);
    }
    __syncwarp();
    for (int i = lane; i < Gv * n; i += 32) {
        const int g = i / n, p = i % n;
        order_out[(g0 + g) * (uint64_t)n + p] = (uint8_t)nib(S.ot[g], p);
    }
}

// ---------------------------------------------------------------------------
// Device-side input validation for the batched host APIs (same rules as the
// host scan in osim_capi.cu: model.py:95-100, engine.py:129-130, unique ids):
// out[0] = lowest offending task index (durations), out[1] = lowest group with
// bad id ranks, out[2] = 1 if any stage is outside the fast range, out[3] = 1
// if any stage is neither null nor in the fast range.
// ---------------------------------------------------------------------------
static __global__ void k_check_batch(const double* __restrict__ durs, const uint8_t* __restrict__ idr,
                                     uint64_t B, int n, uint64_t task0, uint64_t group0,
                                     unsigned long long* __restrict__ out) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    bool notfast = false, notnull = false;
    for (uint64_t b = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; b < B; b += stride) {
        unsigned seen = 0;
        bool badr = false;
        for (int j = 0; j < n; ++j) {
            const double* d = durs + (b * n + j) * 3;
            const double h = d[0], k = d[1], x = d[2];
            const bool ok = h >= 0.0 && k >= 0.0 && x >= 0.0 && h <= 1.7976931348623157e308 &&
                            k <= 1.7976931348623157e308 && x <= 1.7976931348623157e308 &&
                            !(h <= 0 && k <= 0 && x <= 0);
            if (!ok) atomicMin(&out[0], (unsigned long long)(task0 + b * n + j));
            notfast |= !(h >= 0x1p-60 && h < kFastHi && k >= 0x1p-60 && k < kFastHi && x >= 0x1p-60 && x < kFastHi);
            notnull |= !((h == 0.0 || (h >= 0x1p-60 && h < kFastHi)) && (k == 0.0 || (k >= 0x1p-60 && k < kFastHi)) &&
                         (x == 0.0 || (x >= 0x1p-60 && x < kFastHi)));
            if (idr) {
                const unsigned v = idr[b * n + j];
                badr |= v >= (unsigned)n || ((seen >> v) & 1u);
                seen |= 1u << (v & 31u);
            }
        }
        if (badr) atomicMin(&out[1], (unsigned long long)(group0 + b));
    }
    if (__any_sync(kFull, notfast) && (threadIdx.x & 31) == 0) atomicExch(&out[2], 1ull);
    if (__any_sync(kFull, notnull) && (threadIdx.x & 31) == 0) atomicExch(&out[3], 1ull);
}

// ---------------------------------------------------------------------------
// Exact order statistics over makespans kept in HBM (np.median for spaces too
// large for the host).  Positive doubles order like
// their uint64 bit patterns, so the k-th smallest is found digit by digit
// (MSB first): each pass histograms the next kRadixBits bits of the values
// that match the already-fixed prefix.  Lanes of a warp that hit the same bin
// are aggregated with __match_any_sync (makespans share their top bits).
// ---------------------------------------------------------------------------
constexpr int kRadixBits = 11;

// Histogram of the dbits-bit digit below a pbits-bit prefix over the values
// carrying that prefix (bit patterns of positive doubles order like the
// values).  With `out`, the matching values are also appended to out
// (warp-aggregated, order unspecified), so later passes can run on them.
// The global histogram is 64-bit: a digit bin can hold more than 2^32 values
// (13! = 6.2e9 makespans fit one GPU).  The per-block shared counts stay
// 32-bit; a block visits at most ceil(count / (gridDim.x * 256)) * 256
// values, which the launchers keep below 2^32 (radix_grid).
static __global__ void __launch_bounds__(256) k_radix_hist(const unsigned long long* __restrict__ vals,
                                                           uint64_t count, unsigned long long prefix, int pbits,
                                                           int dbits, unsigned long long* __restrict__ hist,
                                                           unsigned long long* __restrict__ out = nullptr,
                                                           unsigned long long* __restrict__ out_count = nullptr) {
    __shared__ unsigned sh[1 << kRadixBits];
    const int nb = 1 << dbits;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    const int shift = 64 - pbits - dbits;
    const unsigned mask = (unsigned)nb - 1u;
    const int lane = threadIdx.x & 31;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t b = (uint64_t)blockIdx.x * blockDim.x; b < count; b += stride) {
        const uint64_t i = b + threadIdx.x;
        const bool valid = i < count;
        const unsigned long long u = valid ? vals[i] : 0ull;
        const bool match = valid && (pbits == 0 || (u >> (64 - pbits)) == prefix);
        const unsigned digit = (unsigned)(u >> shift) & mask;
        OSIM_DCHECK(digit < (unsigned)nb);
        const unsigned key = match ? digit : 0xFFFFFFFFu;
        const unsigned peers = __match_any_sync(kFull, key);
        if (match && lane == __ffs(peers) - 1) atomicAdd(&sh[digit], (unsigned)__popc(peers));
        if (out) {
            const unsigned mm = __ballot_sync(kFull, match);
            if (mm) {
                unsigned long long base = 0;
                if (lane == __ffs(mm) - 1) base = atomicAdd(out_count, (unsigned long long)__popc(mm));
                base = __shfl_sync(kFull, base, __ffs(mm) - 1);
                if (match) out[base + __popc(mm & ((1u << lane) - 1u))] = u;
            }
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nb; i += blockDim.x)
        if (sh[i]) atomicAdd(&hist[i], (unsigned long long)sh[i]);
}

// ---------------------------------------------------------------------------
// Diagnostics
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t splitmix(uint64_t& x) {
    uint64_t z = (x += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static __global__ void k_selftest_div(uint64_t samples, uint64_t seed, unsigned long long* mism) {
    uint64_t st = seed ^ ((uint64_t)(blockIdx.x * blockDim.x + threadIdx.x) * 0x2545F4914F6CDD1Dull);
    unsigned long long bad = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = blockIdx.x * blockDim.x + threadIdx.x; i < samples; i += stride) {
        const uint64_t a = splitmix(st), b = splitmix(st), c = splitmix(st);
        // y: durations / sigma in [2^-60, 2^60] (a superset of the fast range), random mantissa
        int ey = (int)(a % 121) - 60;
        uint64_t my = (b & 0xFFFFFFFFFFFFFull);
        if ((c & 7) == 0) my = 0xFFFFFFFFFFFFFull;
        if ((c & 7) == 1) my = 0;
        const double y = __longlong_as_double(((long long)(1023 + ey) << 52) | (long long)my);
        // x: remaining work: y * fraction, or a raw value of nearby magnitude
        double x;
        const uint64_t d = splitmix(st);
        if ((c >> 3) & 1) {
            const double frac = (double)(d >> 11) * (1.0 / 9007199254740992.0);
            x = __dmul_rn(y, frac);
        } else {
            int ex = ey + (int)((d >> 52) % 140) - 70;
            x = __longlong_as_double(((long long)(1023 + ex) << 52) | (long long)(d & 0xFFFFFFFFFFFFFull));
        }
        if ((c >> 4 & 63) == 0) x = 0.0;
        const double ry = __ddiv_rn(1.0, y);
        if (divq<true>(x, y, ry) != __ddiv_rn(x, y)) ++bad;
    }
    for (int m = 16; m >= 1; m >>= 1) bad += __shfl_xor_sync(kFull, bad, m);
    if ((threadIdx.x & 31) == 0 && bad) atomicAdd(mism, bad);
}

// Adversarial operands for the fast-path division (mode 1 of
// osim_selftest_div_mode): mantissas that sit on rounding boundaries --
// all ones, all ones minus a few ulps, one plus a few ulps, runs of ones --
// for divisor and dividend, exponents placing the quotient on both sides of
// a binade boundary, and dividends that are rounded products y * (1 - 2^-k).
__device__ __forceinline__ uint64_t hard_mant(uint64_t a, uint64_t b) {
    const uint64_t full = 0xFFFFFFFFFFFFFull;
    switch (a & 7) {
        case 0: return full;
        case 1: return full - (b & 0xFFF);
        case 2: return b & 0xFFF;
        case 3: return full & ~((1ull << (b % 52)) - 1ull);  // ones down to bit b % 52
        case 4: return (1ull << (b % 52)) - 1ull;           // ones below bit b % 52
        case 5: return (b & full) | 0xFFFFFull;             // random, low 20 bits set
        case 6: return (b & full) & ~0xFFFFFull;            // random, low 20 bits clear
        default: return b & full;
    }
}

static __global__ void k_selftest_div_hard(uint64_t samples, uint64_t seed, unsigned long long* mism) {
    uint64_t st = seed ^ ((uint64_t)(blockIdx.x * blockDim.x + threadIdx.x) * 0x9E3779B97F4A7C15ull);
    unsigned long long bad = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = blockIdx.x * blockDim.x + threadIdx.x; i < samples; i += stride) {
        const uint64_t a = splitmix(st), b = splitmix(st), c = splitmix(st), d = splitmix(st);
        const int ey = (int)(a % 82) - 60;  // y in [2^-60, 2^22): the fast range of durations
        const double y = __longlong_as_double(((long long)(1023 + ey) << 52) | (long long)hard_mant(a >> 8, b));
        double x;
        if ((c & 3) == 0) {  // a rounded product y * (1 - 2^-k): remaining work just below a duration
            const double frac = 1.0 - __longlong_as_double((long long)(1023 - 1 - (int)(d % 60)) << 52);
            x = __dmul_rn(y, frac);
        } else {
            const int ex = ey + (int)((c >> 2) % 7) - 3 - (((c >> 5) & 7) == 0 ? (int)(d % 40) : 0);
            x = __longlong_as_double(((long long)(1023 + ex) << 52) | (long long)hard_mant(c >> 8, d));
        }
        const double ry = __ddiv_rn(1.0, y);
        if (divq<true>(x, y, ry) != __ddiv_rn(x, y)) ++bad;
    }
    for (int m = 16; m >= 1; m >>= 1) bad += __shfl_xor_sync(kFull, bad, m);
    if ((threadIdx.x & 31) == 0 && bad) atomicAdd(mism, bad);
}

// DFMA throughput: 8 independent chains per thread.
static __global__ void __launch_bounds__(256) k_fp64_peak(double* sink, int iters, double a, double b) {
    double x0 = threadIdx.x * 1e-9, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
    double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
#pragma unroll 1
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            x0 = __fma_rn(x0, a, b); x1 = __fma_rn(x1, a, b); x2 = __fma_rn(x2, a, b);
            x3 = __fma_rn(x3, a, b); x4 = __fma_rn(x4, a, b); x5 = __fma_rn(x5, a, b);
            x6 = __fma_rn(x6, a, b); x7 = __fma_rn(x7, a, b);
        }
    }
    const double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
    if (s == 1234.5678) sink[0] = s;
}

}  // namespace osim
