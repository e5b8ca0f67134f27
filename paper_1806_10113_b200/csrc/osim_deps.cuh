// osim_deps.cuh -- simulator with dependency gates and 1-DMA waves, for the
// NoReorder interleaving distribution (SURVEY.md 8(f) row f1:
// workload.py:259-327) and engine.simulate(..., deps=...).
//
// Queues are explicit per thread (task ids packed 4 bits each), built the
// way DeviceSim.submit builds them (engine.py:115-156), one submit per wave:
// simulate_sequence (workload.py:277-304) splits a 1-DMA sequence into a new
// wave whenever a task's prerequisite sits in the current wave, and each
// submit appends the wave's HtDs and then its DtHs to the shared XFER
// queue.  Readiness adds the deps gate (engine.py:168-171): a command waits
// until its task's prerequisite task has finalized all of its commands.
// Arithmetic is the reference's op sequence with IEEE division (general
// path), so results are bit-identical to the oracle.
#pragma once

#include "osim_kernels.cuh"

namespace osim {

struct Queue32 {  // up to 32 entries: 4-bit task id + 1 kind bit (XFER: 1 = DtH)
    uint64_t t[2];
    uint32_t kind;
    int len;
    __device__ __forceinline__ void clear() { t[0] = t[1] = 0; kind = 0; len = 0; }
    __device__ __forceinline__ void push(int task, int isD) {
        OSIM_DCHECK(len >= 0 && len < 32 && task >= 0 && task < 16);
        t[len >> 4] |= (uint64_t)task << (4 * (len & 15));
        kind |= (uint32_t)isD << len;
        ++len;
    }
    __device__ __forceinline__ int task(int i) const { return (int)((t[i >> 4] >> (4 * (i & 15))) & 0xF); }
    __device__ __forceinline__ int isD(int i) const { return (kind >> i) & 1; }
};

// dep: nibble-packed (prerequisite task + 1) per task id, 0 = none
template <int DMA>
struct DepSim {
    Durs D;
    double sigma;
    Queue32 q[3];  // 2-DMA: 0 HtD, 1 DtH, 2 K;  1-DMA: 0 XFER, 2 K
    int h[3];
    bool run[3];
    int ck[3];     // task of the running command per lane
    int kk[3];     // kind of the running command (0 HtD, 1 K, 2 DtH)
    double rem[3], nd[3];
    double now;
    uint64_t dep;
    unsigned doneH, doneK, doneD;
    int ncmd;

    __device__ __forceinline__ bool nonnull(int k, int t) const { return D.nd(k, t) > 0.0; }
    __device__ __forceinline__ int depof(int t) const { return (int)((dep >> (4 * t)) & 0xF) - 1; }

    // order: packed task ids, len positions; waves: split as simulate_sequence
    __device__ void init(const Durs& d, double sg, uint64_t order, int len, uint64_t dp, bool waves,
                         int ntask) {
        D = d;
        sigma = sg;
        dep = dp;
        now = 0.0;
        for (int l = 0; l < 3; ++l) { q[l].clear(); h[l] = 0; run[l] = false; rem[l] = 1.0; nd[l] = 1.0; }
        doneH = doneK = doneD = 0;
        for (int t = 0; t < ntask; ++t) {  // null stages are done from the start (engine.py:133-135)
            if (!nonnull(0, t)) doneH |= 1u << t;
            if (!nonnull(1, t)) doneK |= 1u << t;
            if (!nonnull(2, t)) doneD |= 1u << t;
        }
        ncmd = 0;
        int w0 = 0;          // first position of the current wave
        unsigned inw = 0;    // tasks of the current wave
        for (int p = 0; p <= len; ++p) {
            const int t = p < len ? nib(order, p) : 0;
            const bool flush = p == len || (DMA == 1 && waves && depof(t) >= 0 && ((inw >> depof(t)) & 1u));
            if (flush) {  // DeviceSim.submit of positions [w0, p)
                for (int i = w0; i < p; ++i) {
                    const int u = nib(order, i);
                    if (nonnull(0, u)) { q[0].push(u, 0); ++ncmd; }
                    if (nonnull(1, u)) { q[2].push(u, 0); ++ncmd; }
                    if (nonnull(2, u) && DMA == 2) { q[1].push(u, 0); ++ncmd; }
                }
                if (DMA == 1)
                    for (int i = w0; i < p; ++i) {
                        const int u = nib(order, i);
                        if (nonnull(2, u)) { q[0].push(u, 1); ++ncmd; }
                    }
                w0 = p;
                inw = 0;
            }
            if (p < len) inw |= 1u << t;
        }
    }

    __device__ __forceinline__ bool finished(int t) const {
        return (((doneH & doneK & doneD) >> t) & 1u) != 0;
    }
    __device__ __forceinline__ bool ready(int kind, int t) const {
        const int pd = depof(t);
        if (pd >= 0 && !finished(pd)) return false;  // engine.py:169-171
        if (kind == 1) return (doneH >> t) & 1u;
        if (kind == 2) return ((doneK & doneH) >> t) & 1u;
        return true;
    }

    __device__ __forceinline__ bool drained() const {
        return h[0] >= q[0].len && h[1] >= q[1].len && h[2] >= q[2].len;
    }

    // returns false when nothing runs and nothing can start (a stall)
    __device__ bool step(TimelineOut* tl) {
        for (int l = 0; l < 3; ++l) {  // engine.py:188-194
            if (run[l] || h[l] >= q[l].len) continue;
            const int t = q[l].task(h[l]);
            const int kind = (l == 2) ? 1 : ((l == 1) ? 2 : (q[l].isD(h[l]) ? 2 : 0));
            if (!ready(kind, t)) continue;
            run[l] = true;
            ck[l] = t;
            kk[l] = kind;
            nd[l] = D.nd(kind, t);
            rem[l] = nd[l];
            if (tl) tl->start[3 * t + kind] = now;
        }
        if (!run[0] && !run[1] && !run[2]) return false;
        const bool ov = DMA == 2 && run[0] && run[1];
        double dt = 0.0;
        bool first = true;
        double rate[3];
        for (int l = 0; l < 3; ++l) {  // engine.py:207-210 (lane order HtD, DtH, K)
            const int ll = (l == 1) ? 1 : l;
            rate[ll] = (ov && ll != 2) ? sigma : 1.0;
        }
        const int order3[3] = {0, 1, 2};
        for (int i = 0; i < 3; ++i) {
            const int l = order3[i];
            if (!run[l]) continue;
            const double v = __ddiv_rn(rem[l], rate[l]);
            if (first || v < dt) dt = v;
            first = false;
        }
        now = __dadd_rn(now, dt);
        for (int l = 0; l < 3; ++l) {
            if (!run[l]) continue;
            const double left = __dsub_rn(rem[l], __dmul_rn(dt, rate[l]));
            rem[l] = __dmul_rn(__ddiv_rn(pymax0(left), nd[l]), nd[l]);
        }
        for (int l = 0; l < 3; ++l) {  // engine.py:216-231
            if (!run[l] || rem[l] > kEndEps) continue;
            run[l] = false;
            ++h[l];
            const int t = ck[l];
            if (kk[l] == 0) doneH |= 1u << t;
            else if (kk[l] == 1) doneK |= 1u << t;
            else doneD |= 1u << t;
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

// M(c - e_w) = M(c) * c_w / |c|: an exact integer below 2^53 (M <= 16!), so
// one correctly rounded FP64 multiply and divide give it exactly -- far
// cheaper than 64-bit integer division.
__device__ __forceinline__ uint64_t mult_next(uint64_t M, int cw, int rem) {
    return (uint64_t)__ddiv_rn(__dmul_rn((double)M, (double)cw), (double)rem);
}

// sorted(set(permutations(labels))) rank -> packed task order (task (w, j) =
// w*N + j): multinomial unranking, M(c - e_w) = M(c) * c_w / |c| exactly.
__device__ __forceinline__ uint64_t unrank_labels(uint64_t r, int T, int N, uint64_t mtotal) {
    int c[16];
    for (int w = 0; w < T; ++w) c[w] = N;
    int rem = T * N;
    uint64_t M = mtotal;
    uint64_t order = 0;
    int cnt[16];
    for (int w = 0; w < T; ++w) cnt[w] = 0;
    for (int p = 0; p < T * N; ++p) {
        for (int w = 0; w < T; ++w) {
            if (!c[w]) continue;
            const uint64_t m = mult_next(M, c[w], rem);
            if (r < m) {
                order |= (uint64_t)(w * N + cnt[w]) << (4 * p);
                ++cnt[w];
                --c[w];
                --rem;
                M = m;
                break;
            }
            r -= m;
        }
    }
    return order;
}

__device__ __forceinline__ uint64_t chain_deps(int T, int N) {
    uint64_t dep = 0;
    for (int w = 0; w < T; ++w)
        for (int j = 1; j < N; ++j) dep |= (uint64_t)(w * N + j) << (4 * (w * N + j));  // (t-1)+1 = t
    return dep;
}

template <int DMA>
__global__ void __launch_bounds__(kBlock) k_interleave(const double* __restrict__ durs, int T, int N, double sigma,
                                                       uint64_t lo, uint64_t hi, uint64_t mtotal, double thr,
                                                       Part* __restrict__ parts, double* __restrict__ ms_out,
                                                       int* __restrict__ err) {
    __shared__ double sd[3 * kStride], sr[3 * kStride];
    __shared__ Part sh[32];
    const int n = T * N;
    stage_durs(durs, n, sd, sr);
    __syncthreads();
    const Durs Dd{sd, sr, 1};
    const uint64_t dep = chain_deps(T, N);
    Part acc;
    part_init(acc);
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t base = lo + (uint64_t)blockIdx.x * blockDim.x; base < hi; base += stride) {
        const uint64_t r = base + threadIdx.x;
        if (r >= hi) continue;
        DepSim<DMA> s;
        s.init(Dd, sigma, unrank_labels(r, T, N, mtotal), n, dep, true, n);
        if (!s.run_all()) atomicExch(err, OSIM_ESTALL);
        part_add<true>(acc, s.now, r, thr);
        if (ms_out) ms_out[r - lo] = s.now;
    }
    acc = block_reduce(acc, sh);
    if (threadIdx.x == 0) parts[blockIdx.x] = acc;
}

// 1-DMA NoReorder fast path.  simulate_sequence (workload.py:277-304) cuts
// the sequence into waves -- a task whose prerequisite (the same worker's
// previous task) sits in the current wave opens a new one -- and each submit
// appends the wave's HtDs, then its DtHs, to the XFER queue; the K queue
// keeps sequence order.  With a wave [a, b) the XFER slot of HtD(p) is
// p + a and of DtH(p) is p + b.  A prerequisite always lies in an earlier
// wave, whose DtH block the XFER lane has passed before this wave's HtDs,
// so the deps gate never binds; readiness is K(p): XFER slot count > p +
// ws(p); XFER DtH(p): K head > p.  Every stage non-null and in the FastSim
// range; same op sequence as DepSim.
template <bool PRE>
struct WaveSim {
    uint32_t base;
    uint64_t seq;
    uint64_t wsq, weq;  // per position: wave start, wave end - 1 (nibbles)
    int n4;
    double now, r0, r2, d0, d2, c0, c2;
    int x;       // 4 * XFER slots finalized
    int p0, h0;  // XFER current position and kind (0 HtD, 1 DtH)
    int s2;      // 4 * K head position

    __device__ __forceinline__ void init(uint32_t b, uint64_t sq, int n, uint64_t ws, uint64_t we) {
        base = b;
        seq = PRE ? (sq << 4) : sq;
        wsq = ws;
        weq = we;
        n4 = 4 * n;
        now = 0.0;
        r0 = r2 = kBig;
        d0 = d2 = c0 = c2 = 1.0;
        x = 0;
        p0 = 0;
        h0 = 0;
        s2 = 0;
    }
    __device__ __forceinline__ int wsof(int p) const { return (int)((wsq >> (4 * p)) & 0xF); }
    __device__ __forceinline__ int weof(int p) const { return (int)((weq >> (4 * p)) & 0xF) + 1; }

    __device__ __forceinline__ void step() {
        const bool st0 = idle(r0) && x < 2 * n4 && (h0 == 0 || s2 > 4 * p0);
        const bool st2 = idle(r2) && s2 < n4 && x > 4 * ((s2 >> 2) + wsof(s2 >> 2));
        start_if(st0, base + (h0 ? 512u : 0u) + task_off<PRE>(seq, 4 * p0), d0, c0, r0);
        start_if(st2, base + 256 + task_off<PRE>(seq, s2), d2, c2, r2);
        const double dt = dmin(r0, r2);  // no overlap on one DMA engine: rate 1
        now = __dadd_rn(now, dt);
        r0 = __dmul_rn(divq<true>(__dsub_rn(r0, dt), d0, c0), d0);
        r2 = __dmul_rn(divq<true>(__dsub_rn(r2, dt), d2, c2), d2);
        const bool f0 = r0 <= kEndEps;
        r0 = retire_or_drain(f0, r0, x + 4 >= 2 * n4);
        if (f0) {
            x += 4;
            const int e = weof(p0);
            if (p0 + 1 < e) ++p0;
            else if (h0 == 0) { h0 = 1; p0 = wsof(p0); }
            else { h0 = 0; p0 = e; }
        }
        if (r2 <= kEndEps) { r2 = retire(r2); s2 += 4; }
    }
    __device__ __forceinline__ bool drained() const { return x >= 2 * n4; }
};

// ---------------------------------------------------------------------------
// Prefix sharing for the NoReorder distribution.  Interleavings are ranked in
// lexicographic order of their worker-label sequences, so a run of K
// consecutive ranks [r0, r0 + K) shares the first M = lcp(seq(r0),
// seq(r0 + K - 1)) labels -- the same M tasks, the same prerequisites.  Up to
// the step in which HtD(M - 1) finalizes no command of a position >= M can
// have started (the HtD lane is a FIFO; K(p) waits for HtD(p), DtH(p) for
// K(p); the deps gate only delays starts), so that state is common to the
// whole run: each thread simulates it once, stores it in its shared-memory
// slot and replays the K suffixes from it, stepping to the next sequence by
// a multiset next-permutation of the label suffix (no per-rank unranking).
// Per-sequence operation sequences are unchanged, so makespans are
// bit-identical to DepSim's (FastSim with the prerequisite gate on the HtD
// start: with every stage non-null a task is finished exactly when its DtH
// finalized, and DtHs finalize in sequence order).
// ---------------------------------------------------------------------------
__device__ __forceinline__ int lab_at(uint64_t lab, int p) { return (int)((lab >> (4 * p)) & 0xF); }

// labels of rank r (multinomial unranking, as unrank_labels)
__device__ __forceinline__ uint64_t unrank_lab(uint64_t r, int T, int N, uint64_t mtotal) {
    int c[16];
    for (int w = 0; w < T; ++w) c[w] = N;
    int rem = T * N;
    uint64_t M = mtotal, lab = 0;
    for (int p = 0; p < T * N; ++p) {
        for (int w = 0; w < T; ++w) {
            if (!c[w]) continue;
            const uint64_t m = mult_next(M, c[w], rem);
            if (r < m) {
                lab |= (uint64_t)w << (4 * p);
                --c[w];
                --rem;
                M = m;
                break;
            }
            r -= m;
        }
    }
    return lab;
}

// next sequence in lexicographic order (std::next_permutation on a multiset);
// the pivot lies at a position >= the run's common prefix
__device__ __forceinline__ uint64_t lab_next(uint64_t lab, int n) {
    int i = n - 2;
    while (i >= 0 && lab_at(lab, i) >= lab_at(lab, i + 1)) --i;
    if (i < 0) return lab;
    const int a = lab_at(lab, i);
    int j = n - 1;
    while (lab_at(lab, j) <= a) --j;
    const int b = lab_at(lab, j);
    lab = (lab & ~(0xFull << (4 * i)) & ~(0xFull << (4 * j))) | ((uint64_t)b << (4 * i)) | ((uint64_t)a << (4 * j));
    // reverse positions i+1 .. n-1
    uint64_t out = lab & ((i + 1 >= 16) ? ~0ull : ((1ull << (4 * (i + 1))) - 1ull));
    for (int p = i + 1, q = n - 1; p < n; ++p, --q) out |= (uint64_t)lab_at(lab, q) << (4 * p);
    return out;
}

// task order and packed prerequisites (1 + position of the worker's previous
// task) of positions [M, n), from the counters of the prefix [0, M)
__device__ __forceinline__ void lab_tasks(uint64_t lab, int N, int M, int n, uint64_t cnt, uint64_t last,
                                          uint64_t& order, uint64_t& dseq) {
    const uint64_t keep = (M >= 16) ? ~0ull : ((1ull << (4 * M)) - 1ull);
    order &= keep;
    dseq &= keep;
    for (int p = M; p < n; ++p) {
        const int w = lab_at(lab, p), sh = 4 * w;
        const int c = (int)((cnt >> sh) & 0xF);
        order |= (uint64_t)(w * N + c) << (4 * p);
        dseq |= ((last >> sh) & 0xFull) << (4 * p);
        cnt += 1ull << sh;
        last = (last & ~(0xFull << sh)) | ((uint64_t)((p + 1) & 0xF) << sh);
    }
}

// Runs are sorted by phase-A step count within the CTA before the replays
// (a deterministic counting sort, as pfx_sort): a warp's replays run for
// 3n - min(sa) steps, and unsorted runs mix common prefixes of very
// different lengths.
#ifndef OSIM_F1_MINB
#define OSIM_F1_MINB 3
#endif
struct RunSort {
    int cnt[kNW][kSaBins];
    int base[kSaBins];
    short order[kBlock];
    uint64_t lab[kBlock], r0[kBlock];
    int m[kBlock], sa[kBlock];  // m: M | valid << 8
};

__device__ __forceinline__ int run_sort(RunSort& S, int key) {
    const int ti = threadIdx.x, lane = ti & 31, w = ti >> 5;
    for (int i = lane; i < kSaBins; i += 32) S.cnt[w][i] = 0;
    __syncwarp();
    const unsigned m = __match_any_sync(kFull, key);
    if (lane == __ffs(m) - 1) S.cnt[w][key] = __popc(m);
    __syncthreads();
    if (w == 0) {
        int carry = 0;
#pragma unroll
        for (int b0 = 0; b0 < kSaBins; b0 += 32) {
            const int b = b0 + lane;
            int t = 0;
#pragma unroll
            for (int ww = 0; ww < kNW; ++ww) t += S.cnt[ww][b];
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
    int r = S.base[key] + __popc(m & ((1u << lane) - 1u));
    for (int ww = 0; ww < w; ++ww) r += S.cnt[ww][key];
    S.order[r] = (short)ti;
    __syncthreads();
    return S.order[ti];
}

// first and last rank of this thread's run, its labels and common prefix
__device__ __forceinline__ void run_open(uint64_t run, uint64_t runs, uint64_t lo, uint64_t hi, int K, int T, int N,
                                         uint64_t mtotal, uint64_t& r0, uint64_t& lab, int& M) {
    const int n = T * N;
    r0 = lo + (run < runs ? run : 0) * (uint64_t)K;
    const uint64_t r1 = (r0 + (uint64_t)K < hi) ? r0 + (uint64_t)K : hi;
    lab = unrank_lab(r0, T, N, mtotal);
    const uint64_t x = lab ^ unrank_lab(r1 - 1, T, N, mtotal);
    M = x ? (__ffsll((long long)x) - 1) >> 2 : n;
}

// task order, prerequisites and the prefix counters (occurrences, 1 + last
// position per worker) of a run's first sequence
__device__ __forceinline__ void run_tasks(uint64_t lab, int N, int M, int n, uint64_t& cnt, uint64_t& last,
                                          uint64_t& order, uint64_t& dseq) {
    cnt = last = order = dseq = 0;
    lab_tasks(lab, N, 0, n, 0, 0, order, dseq);
    for (int p = 0; p < M; ++p) {
        const int sh4 = 4 * lab_at(lab, p);
        cnt += 1ull << sh4;
        last = (last & ~(0xFull << sh4)) | ((uint64_t)((p + 1) & 0xF) << sh4);
    }
}

#ifndef OSIM_F1_LEAN
#define OSIM_F1_LEAN 1
#endif
template <bool SIGP2, bool PRE>
__global__ void __launch_bounds__(kBlock, OSIM_F1_MINB) k_interleave_pfx(const double* __restrict__ durs, int T, int N,
                                                           double sigma, uint64_t lo, uint64_t hi, uint64_t mtotal,
                                                           int K, double thr, Part* __restrict__ parts,
                                                           double* __restrict__ ms_out, int* __restrict__ err) {
    __shared__ double2 sdr[3 * kStride];
    __shared__ Part sh[32];
    __shared__ CkSlots<1> ck;
    __shared__ RunSort S;
    const int n = T * N;
    stage_dr(durs, n, sdr);
    __syncthreads();
    const uint32_t base = opaque_u32((uint32_t)__cvta_generic_to_shared(sdr));  // kept in a register
    const double rsig = __ddiv_rn(1.0, sigma);
    const int ti = threadIdx.x;
    Part acc;
    part_init(acc);
    const uint64_t runs = (hi - lo + (uint64_t)K - 1) / (uint64_t)K;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t b0 = (uint64_t)blockIdx.x * blockDim.x; b0 < runs; b0 += stride) {
        __syncthreads();  // the previous round's slots have been read
        // ---- phase A: this thread's run to its common-prefix checkpoint
        {
            const uint64_t run = b0 + ti;
            uint64_t r0, lab, cnt, last, order, dseq;
            int M;
            run_open(run, runs, lo, hi, K, T, N, mtotal, r0, lab, M);
            run_tasks(lab, N, M, n, cnt, last, order, dseq);
            FastSim<2, SIGP2, false, PRE, true> s;
            s.init(base, order, n);
            s.dseq = PRE ? (dseq << 4) : dseq;
            const int sa = advance_to(s, M, sigma, rsig);
            ck_store(ck, 0, ti, s);
            const bool valid = run < runs;
            S.lab[ti] = lab;
            S.r0[ti] = r0;
            S.m[ti] = M | (valid ? 256 : 0);
            S.sa[ti] = valid ? sa : kSaBins - 1;
        }
        // ---- reassign by sa, then replay the taken run's sequences
        const int e = run_sort(S, S.sa[ti]);
        const uint64_t r0 = S.r0[e];
        uint64_t lab = S.lab[e];
        const int M = S.m[e] & 255;
        const bool valid = (S.m[e] >> 8) != 0;
        const uint64_t r1 = (r0 + (uint64_t)K < hi) ? r0 + (uint64_t)K : hi;
        uint64_t cnt, last, order, dseq;
        run_tasks(lab, N, M, n, cnt, last, order, dseq);
        const int rest = 3 * n - __reduce_min_sync(kFull, valid ? S.sa[e] : 3 * n);
        FastSim<2, SIGP2, false, PRE, true> s;
        s.init(base, order, n);
#pragma unroll 1
        for (int q = 0; q < K; ++q) {
            if (q > 0) {
                lab = lab_next(lab, n);
                lab_tasks(lab, N, M, n, cnt, last, order, dseq);
            }
            ck_load(ck, 0, e, s, M);
            s.set_seq(order);
            s.dseq = PRE ? (dseq << 4) : dseq;
#if OSIM_F1_LEAN
            s.template run_phased<true, SIGP2 ? OSIM_PH_FULL_P2 : OSIM_PH_FULL>(rest, sigma, rsig);
            const uint64_t r = r0 + (uint64_t)q;
            if (valid && r < r1) {
                if (!s.drained()) atomicExch(err, OSIM_ESTALL);
                leaf_add<true>(acc, s.now, r, thr);  // the prefix kernels' leaf (see there)
                acc.count += 1;
                if (ms_out) ms_out[r - lo] = s.now;
            }
            // exponent split-off every 8 sequences (fast-path makespans: see pfx_leaves)
            if ((q & 7) == 7 || q == K - 1) renorm<false>(acc.lpm, acc.lpe);
#else
            s.run_phased(rest, sigma, rsig);
            const uint64_t r = r0 + (uint64_t)q;
            if (valid && r < r1) {
                if (!s.drained()) atomicExch(err, OSIM_ESTALL);
                part_add<true>(acc, s.now, r, thr);
                if (ms_out) ms_out[r - lo] = s.now;
            }
#endif
        }
    }
    acc = block_reduce(acc, sh);
    if (threadIdx.x == 0) parts[blockIdx.x] = acc;
}

// 1-DMA runs.  The wave split of a sequence is fixed on the common prefix
// except for where its last wave ends (that depends on the label at M), so
// the checkpoint keeps the clock, the K lane and the XFER slot count, and
// each sequence recomputes its waves and, from them, the XFER item that
// follows HtD(M - 1): HtD(M) when M is inside that wave, else the wave's
// DtH block.
__device__ __forceinline__ void lab_waves(uint64_t lab, int n, uint64_t& wsq, uint64_t& weq) {
    unsigned starts = 0;
    uint64_t last = 0;  // 1 + last position per worker
    int w0 = 0;
    for (int p = 0; p < n; ++p) {
        const int sh = 4 * lab_at(lab, p);
        const int lp = (int)((last >> sh) & 0xF) - 1;
        if (p == 0 || lp >= w0) { starts |= 1u << p; w0 = p; }
        last = (last & ~(0xFull << sh)) | ((uint64_t)((p + 1) & 0xF) << sh);
    }
    wsq = weq = 0;
    int ws = 0;
    for (int p = 0; p < n; ++p) {
        if ((starts >> p) & 1u) ws = p;
        const unsigned after = starts & ~((2u << p) - 1u);
        const int we = after ? __ffs(after) - 1 : n;
        wsq |= (uint64_t)ws << (4 * p);
        weq |= (uint64_t)(we - 1) << (4 * p);
    }
}

// Waves of the run's later sequences: the wave starts below M are the run's
// (prefix-determined), so only positions >= M extend the start set and only
// the ws / we nibbles from the wave holding position M - 1 on change.
// startsM / w0M / lastM: start bits below M, start of the wave holding M - 1,
// 1 + last position per worker over the prefix (lab_wave_prefix).
__device__ __forceinline__ void lab_wave_prefix(uint64_t lab, int M, unsigned& starts, int& w0, uint64_t& last) {
    starts = 0;
    w0 = 0;
    last = 0;
    for (int p = 0; p < M; ++p) {
        const int sh = 4 * lab_at(lab, p);
        const int lp = (int)((last >> sh) & 0xF) - 1;
        if (p == 0 || lp >= w0) { starts |= 1u << p; w0 = p; }
        last = (last & ~(0xFull << sh)) | ((uint64_t)((p + 1) & 0xF) << sh);
    }
}

__device__ __forceinline__ void lab_waves_from(uint64_t lab, int n, int M, unsigned startsM, int w0M, uint64_t lastM,
                                               uint64_t& wsq, uint64_t& weq) {
    unsigned starts = startsM;
    int w0 = w0M;
    uint64_t last = lastM;
    for (int p = M; p < n; ++p) {
        const int sh = 4 * lab_at(lab, p);
        const int lp = (int)((last >> sh) & 0xF) - 1;
        if (p == 0 || lp >= w0) { starts |= 1u << p; w0 = p; }
        last = (last & ~(0xFull << sh)) | ((uint64_t)((p + 1) & 0xF) << sh);
    }
    const uint64_t keep = (w0M >= 16) ? ~0ull : ((1ull << (4 * w0M)) - 1ull);
    wsq &= keep;
    weq &= keep;
    int ws = w0M;
    for (int p = w0M; p < n; ++p) {
        if ((starts >> p) & 1u) ws = p;
        const unsigned after = starts & ~((2u << p) - 1u);
        const int we = after ? __ffs(after) - 1 : n;
        wsq |= (uint64_t)ws << (4 * p);
        weq |= (uint64_t)(we - 1) << (4 * p);
    }
}

template <bool PRE>
__global__ void __launch_bounds__(kBlock, OSIM_F1_MINB) k_interleave_pfx1(const double* __restrict__ durs, int T, int N,
                                                            uint64_t lo, uint64_t hi, uint64_t mtotal, int K,
                                                            double thr, Part* __restrict__ parts,
                                                            double* __restrict__ ms_out, int* __restrict__ err) {
    __shared__ double2 sdr[3 * kStride];
    __shared__ Part sh[32];
    __shared__ double cv[4][kBlock];  // now, r2, d2, c2
    __shared__ int cx[2][kBlock];     // x, s2
    __shared__ RunSort S;
    const int n = T * N;
    stage_dr(durs, n, sdr);
    __syncthreads();
    const uint32_t base = opaque_u32((uint32_t)__cvta_generic_to_shared(sdr));  // kept in a register
    const int ti = threadIdx.x;
    Part acc;
    part_init(acc);
    const uint64_t runs = (hi - lo + (uint64_t)K - 1) / (uint64_t)K;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t b0 = (uint64_t)blockIdx.x * blockDim.x; b0 < runs; b0 += stride) {
        __syncthreads();  // the previous round's slots have been read
        {
            const uint64_t run = b0 + ti;
            uint64_t r0, lab, cnt, last, order, dseq, wsq, weq;
            int M;
            run_open(run, runs, lo, hi, K, T, N, mtotal, r0, lab, M);
            run_tasks(lab, N, M, n, cnt, last, order, dseq);
            lab_waves(lab, n, wsq, weq);
            WaveSim<PRE> s;
            s.init(base, order, n, wsq, weq);
            // phase A: to the finalize of HtD(M - 1) = XFER slot M - 1 + ws(M - 1)
            const int xt = (M > 0) ? 4 * (M + s.wsof(M - 1)) : 0;
            int sa = 0;
#pragma unroll 1
            while (__any_sync(kFull, s.x < xt && sa < 3 * kMaxN)) {
                if (s.x < xt && sa < 3 * kMaxN) {
                    s.step();
                    ++sa;
                }
            }
            cv[0][ti] = s.now; cv[1][ti] = s.r2; cv[2][ti] = s.d2; cv[3][ti] = s.c2;
            cx[0][ti] = s.x; cx[1][ti] = s.s2;
            const bool valid = run < runs;
            S.lab[ti] = lab;
            S.r0[ti] = r0;
            S.m[ti] = M | (valid ? 256 : 0);
            S.sa[ti] = valid ? sa : kSaBins - 1;
        }
        const int e = run_sort(S, S.sa[ti]);
        const uint64_t r0 = S.r0[e];
        uint64_t lab = S.lab[e];
        const int M = S.m[e] & 255;
        const bool valid = (S.m[e] >> 8) != 0;
        const uint64_t r1 = (r0 + (uint64_t)K < hi) ? r0 + (uint64_t)K : hi;
        uint64_t cnt, last, order, dseq, wsq, weq, wlast;
        run_tasks(lab, N, M, n, cnt, last, order, dseq);
        unsigned wstarts;
        int w0M;
        lab_wave_prefix(lab, M, wstarts, w0M, wlast);
        lab_waves(lab, n, wsq, weq);
        const int rest = 3 * n - __reduce_min_sync(kFull, valid ? S.sa[e] : 3 * n);
        WaveSim<PRE> s;
#pragma unroll 1
        for (int q = 0; q < K; ++q) {
            if (q > 0) {
                lab = lab_next(lab, n);
                lab_tasks(lab, N, M, n, cnt, last, order, dseq);
                lab_waves_from(lab, n, M, wstarts, w0M, wlast, wsq, weq);
            }
            s.init(base, order, n, wsq, weq);
            s.now = cv[0][e]; s.r2 = cv[1][e]; s.d2 = cv[2][e]; s.c2 = cv[3][e];
            s.x = cx[0][e]; s.s2 = cx[1][e];
            if (M > 0) {  // the XFER item after HtD(M - 1)
                if (M < s.weof(M - 1)) { s.p0 = M; s.h0 = 0; }
                else { s.p0 = s.wsof(M - 1); s.h0 = 1; }
            }
#pragma unroll 1
            for (int st = 0; st < rest; st += 2) {
                s.step();
                s.step();
            }
            const uint64_t r = r0 + (uint64_t)q;
            if (valid && r < r1) {
                if (!s.drained()) atomicExch(err, OSIM_ESTALL);
                part_add<true>(acc, s.now, r, thr);
                if (ms_out) ms_out[r - lo] = s.now;
            }
        }
    }
    acc = block_reduce(acc, sh);
    if (threadIdx.x == 0) parts[blockIdx.x] = acc;
}

template <int DMA>
__global__ void __launch_bounds__(kBlock) k_eval_labels(const double* __restrict__ durs, int T, int N, double sigma,
                                                        const uint8_t* __restrict__ labels, uint64_t cnt,
                                                        Part* __restrict__ parts, double* __restrict__ ms_out,
                                                        int* __restrict__ err) {
    __shared__ double sd[3 * kStride], sr[3 * kStride];
    __shared__ Part sh[32];
    const int n = T * N;
    stage_durs(durs, n, sd, sr);
    __syncthreads();
    const Durs Dd{sd, sr, 1};
    const uint64_t dep = chain_deps(T, N);
    Part acc;
    part_init(acc);
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += stride) {
        int c[16];
        for (int w = 0; w < T; ++w) c[w] = 0;
        uint64_t order = 0;
        for (int p = 0; p < n; ++p) {
            const int w = labels[i * n + p];
            order |= (uint64_t)(w * N + c[w]++) << (4 * p);
        }
        DepSim<DMA> s;
        s.init(Dd, sigma, order, n, dep, true, n);
        if (!s.run_all()) atomicExch(err, OSIM_ESTALL);
        part_add<true>(acc, s.now, i, -kBig);
        ms_out[i] = s.now;
    }
    acc = block_reduce(acc, sh);
    if (threadIdx.x == 0) parts[blockIdx.x] = acc;
}

// engine.simulate(tasks, profile, deps) / workload.simulate_sequence: one
// ordering with an explicit dep array and optional 1-DMA waves.
template <int DMA>
__global__ void k_timeline_dep(const double* __restrict__ durs, int n, double sigma,
                               const uint8_t* __restrict__ order, const int8_t* __restrict__ dep, int waves,
                               double* start, double* end, double* res, int* err) {
    __shared__ double sd[3 * kStride], sr[3 * kStride];
    stage_durs(durs, n, sd, sr);
    __syncthreads();
    if (threadIdx.x != 0) return;
    for (int i = 0; i < 3 * n; ++i) { start[i] = -1.0; end[i] = -1.0; }
    uint64_t seq = 0, dp = 0;
    for (int j = 0; j < n; ++j) seq |= (uint64_t)(order[j] & 0xF) << (4 * j);
    for (int t = 0; t < n; ++t)
        if (dep && dep[t] >= 0) dp |= (uint64_t)(dep[t] + 1) << (4 * t);
    DepSim<DMA> s;
    s.init(Durs{sd, sr, 1}, sigma, seq, n, dp, waves != 0, n);
    TimelineOut tl{start, end};
    if (!s.run_all(&tl)) { *err = OSIM_ESTALL; return; }
    res[0] = s.now;
    // idle_report (engine.py:68-80): spans of a kind sorted by (start, end)
    for (int k = 0; k < 3; ++k) {
        double idle = 0.0, prev_end = 0.0;
        int done = 0;
        for (int it = 0; it < n; ++it) {  // selection in (start, end) order
            int best = -1;
            for (int t = 0; t < n; ++t) {
                const double st = start[3 * t + k];
                if (st < 0.0 || ((done >> t) & 1)) continue;
                if (best < 0 || st < start[3 * best + k] ||
                    (st == start[3 * best + k] && end[3 * t + k] < end[3 * best + k]))
                    best = t;
            }
            if (best < 0) break;
            const double st = start[3 * best + k];
            if (it > 0 && st > prev_end) idle = __dadd_rn(idle, __dsub_rn(st, prev_end));
            prev_end = end[3 * best + k];
            done |= 1 << best;
        }
        res[1 + k] = idle;
    }
}

}  // namespace osim
