// osim_micro.cuh -- the micro-step validation oracle on the GPU (SURVEY.md
// 8(f) row f4): oracle.micro_simulate's fixed-dt tick loop
// (/root/reference/pkg/src/offsim/_micro.py:19-143), one thread per ordering,
// for `offsim validate`-style sweeps (cli.py:162-181).  Every command runs
// only at its queue head and never pauses once started, so a lane's
// remaining work is reset to the nominal duration when its head advances.
// Same per-tick op sequence as the reference (rem -= dt*rate; t = step*dt).
#pragma once

#include "osim_kernels.cuh"

namespace osim {

constexpr double kMicroTol = 1e-9;  // _micro.py:16
constexpr long long kMicroBurst = 1ll << 20;  // ticks per inner burst (runaway bound granularity)

template <int DMA>
struct MicroSim {
    Durs D;
    uint64_t seq;
    int n;
    unsigned nullH, nullK, nullD;
    unsigned doneH, doneK, doneD;
    int hh, hd, hk;
    double rh, rd, rk;
    double t, ms;
    long long step;
    long long ticks;  // ticks executed (the caller's runaway bound)

    __device__ __forceinline__ int skip(int p, unsigned nm) const {
        while (p < n && ((nm >> nib(seq, p)) & 1u)) ++p;
        return p;
    }
    __device__ __forceinline__ void init(const Durs& d, uint64_t s, int nn) {
        D = d;
        seq = s;
        n = nn;
        nullH = nullK = nullD = 0;
        for (int i = 0; i < n; ++i) {
            const int t = nib(seq, i);
            if (!(D.nd(0, t) > 0.0)) nullH |= 1u << t;
            if (!(D.nd(1, t) > 0.0)) nullK |= 1u << t;
            if (!(D.nd(2, t) > 0.0)) nullD |= 1u << t;
        }
        doneH = nullH; doneK = nullK; doneD = nullD;
        hh = skip(0, nullH); hd = skip(0, nullD); hk = skip(0, nullK);
        rh = hh < n ? D.nd(0, nib(seq, hh)) : 0.0;
        rd = hd < n ? D.nd(2, nib(seq, hd)) : 0.0;
        rk = hk < n ? D.nd(1, nib(seq, hk)) : 0.0;
        t = 0.0;
        ms = 0.0;
        step = 0;
        ticks = 0;
    }

    // one tick; false once nothing can execute (the loop's break)
    __device__ __forceinline__ bool tick(double sigma, double dt, TimelineOut* tl) {
        const bool eh = hh < n;
        bool ed = false;
        if (hd < n && (DMA == 2 || !eh)) {  // 1-DMA: DtHs only after every HtD drained
            const int i = nib(seq, hd);
            ed = ((doneK & doneH) >> i) & 1u;
        }
        const bool ek = hk < n && ((doneH >> nib(seq, hk)) & 1u);
        if (!eh && !ed && !ek) return false;
        const double rate = (DMA == 2 && eh && ed) ? sigma : 1.0;
        if (tl) {
            if (eh && tl->start[3 * nib(seq, hh) + 0] < 0.0) tl->start[3 * nib(seq, hh) + 0] = t;
            if (ed && tl->start[3 * nib(seq, hd) + 2] < 0.0) tl->start[3 * nib(seq, hd) + 2] = t;
            if (ek && tl->start[3 * nib(seq, hk) + 1] < 0.0) tl->start[3 * nib(seq, hk) + 1] = t;
        }
        // Ticks up to the next finalization: the enabled lanes and the rate
        // only change when a command finalizes, and t = step * dt is read
        // only then, so the reference's per-tick `rem -= dt * rate` runs in a
        // tight loop (same operations on the same values, tick by tick).
        const double xt = __dmul_rn(dt, rate);
        const double big = 0x1p1000;  // a lane that is not executing never finalizes
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
            const int i = nib(seq, hh);
            if (tl) tl->end[3 * i + 0] = t;
            doneH |= 1u << i;
            hh = skip(hh + 1, nullH);
            if (hh < n) rh = D.nd(0, nib(seq, hh));
            ms = t;
        }
        if (ed && rd <= kMicroTol) {
            const int i = nib(seq, hd);
            if (tl) tl->end[3 * i + 2] = t;
            doneD |= 1u << i;
            hd = skip(hd + 1, nullD);
            if (hd < n) rd = D.nd(2, nib(seq, hd));
            ms = t;
        }
        if (ek && rk <= kMicroTol) {
            const int i = nib(seq, hk);
            if (tl) tl->end[3 * i + 1] = t;
            doneK |= 1u << i;
            hk = skip(hk + 1, nullK);
            if (hk < n) rk = D.nd(1, nib(seq, hk));
            ms = t;
        }
        return true;
    }
};

template <int DMA>
__global__ void __launch_bounds__(kBlock) k_micro(const double* __restrict__ durs, int n, double sigma, double dt,
                                                  uint64_t lo, uint64_t hi, long long max_ticks,
                                                  double* __restrict__ ms_out, int* __restrict__ err) {
    __shared__ double sd[3 * kStride], sr[3 * kStride];
    stage_durs(durs, n, sd, sr);
    __syncthreads();
    const uint64_t r = lo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= hi) return;
    MicroSim<DMA> s;
    s.init(Durs{sd, sr, 1}, unrank_rt(r, n), n);
    while (s.tick(sigma, dt, nullptr))
        if (s.ticks > max_ticks) { atomicExch(err, OSIM_ESTALL); break; }
    ms_out[r - lo] = s.ms;
}

template <int DMA>
__global__ void k_micro_timeline(const double* __restrict__ durs, int n, double sigma, double dt,
                                 const uint8_t* __restrict__ order, long long max_ticks, double* start, double* end,
                                 double* res, int* err) {
    __shared__ double sd[3 * kStride], sr[3 * kStride];
    stage_durs(durs, n, sd, sr);
    __syncthreads();
    if (threadIdx.x != 0) return;
    for (int i = 0; i < 3 * n; ++i) { start[i] = -1.0; end[i] = -1.0; }
    uint64_t seq = 0;
    for (int j = 0; j < n; ++j) seq |= (uint64_t)(order[j] & 0xF) << (4 * j);
    MicroSim<DMA> s;
    s.init(Durs{sd, sr, 1}, seq, n);
    TimelineOut tl{start, end};
    while (s.tick(sigma, dt, &tl))
        if (s.ticks > max_ticks) { *err = OSIM_ESTALL; return; }
    res[0] = s.ms;
}

}  // namespace osim
