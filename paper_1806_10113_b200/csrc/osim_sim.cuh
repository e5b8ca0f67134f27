// osim_sim.cuh -- register-resident FP64 event loop of the temporal
// execution model, one simulation per thread.
//
// This is the B200 formulation of DeviceSim.step/run/timeline
// (/root/reference/pkg/src/offsim/engine.py:182-249).  Instead of command
// objects in per-lane FIFO lists, a thread keeps, per lane, the head
// position in its ordering (a packed 4-bit-per-position sequence), a
// running flag and the running command's remaining work `rem` = rw*nd
// plus its nominal duration `nd` and 1/nd.  Durations live in shared
// memory as kind-major [3][stride] arrays, so every lookup of a task's
// stage is conflict-free (<=16 doubles per kind = one 128-byte bank row).
//
// Operation order is the reference's (engine.py:207-222), all IEEE double
// with explicit round-to-nearest intrinsics so nothing is contracted:
//   cand_c = rem_c / rate_c                       (engine.py:210)
//   dt     = min_c cand_c ;  now = now + dt        (:210-211)
//   left_c = rem_c - dt * rate_c                   (:213)
//   rw_c   = max(left_c, 0.0) / nd_c               (:214)
//   rem_c  = rw_c * nd_c ;  finalize if rem_c <= 1e-9   (:222)
// `rem_c` is exactly the product the reference recomputes at the top of
// the next step, so it is carried instead of rw.
//
// Division.  The fast path divides with Markstein's correction from a
// correctly rounded reciprocal (q0 = x*r, e = fma(-q0, y, x),
// q = fma(e, r, q0)), which returns the correctly rounded quotient for
// operands whose quotient and remainder stay clear of the subnormal range;
// the host only selects it when every duration and sigma lies in
// [2^-60, 2^22) (see kFastHi and osim_capi.cu), and the GPU self-test compares it with
// IEEE division.  The general path (null stages, out-of-range inputs)
// uses IEEE division (__ddiv_rn).
#pragma once

#include <cstdint>
#include <cstdio>

// Device-side bounds and invariant checks, compiled in only for the
// checking build (python -m paper_1806_10113_b200._build --variant dcheck
// -DOSIM_DEBUG_CHECKS; tools/dcheck_run.py).  compute-sanitizer is not
// available on the GPU pool, so shared-memory / global indices and the
// kernels' own invariants are asserted in the code: a violation prints the
// site and traps (the launch fails with cudaErrorLaunchFailure).
#ifdef OSIM_DEBUG_CHECKS
#define OSIM_DCHECK(cond)                                                                          \
    do {                                                                                           \
        if (!(cond)) {                                                                             \
            printf("OSIM_DCHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__, \
                   (int)blockIdx.x, (int)threadIdx.x);                                             \
            __trap();                                                                              \
        }                                                                                          \
    } while (0)
#else
#define OSIM_DCHECK(cond) \
    do {                  \
    } while (0)
#endif

namespace osim {

constexpr double kEndEps = 1e-9;  // engine.py:26 _END_EPS
#ifndef OSIM_CEPS
#define OSIM_CEPS 1
#endif
#if OSIM_CEPS
// the same value in the constant bank: FastSim's finalize compares take it as
// a direct operand instead of rematerializing it in the replay loops
static __constant__ double c_end_eps = 1e-9;
#define OSIM_FIN_EPS c_end_eps
#else
#define OSIM_FIN_EPS kEndEps
#endif

#ifndef OSIM_PH_FULL
#define OSIM_PH_FULL 2  // FastSim::run_phased (2-DMA): steps per phase vote, full / K+DtH phases
#endif
#ifndef OSIM_PH_KD
#define OSIM_PH_KD 2
#endif
#ifndef OSIM_PH_FULL_P2
#define OSIM_PH_FULL_P2 3  // the prefix kernels' full phase at power-of-two sigma, n >= 10
#endif
#ifndef OSIM_EXPSHIFT
#define OSIM_EXPSHIFT 1  // FastSim, power-of-two sigma: rate factors as exponent shifts (see step())
#endif

// Step bounds.  The command that sets dt leaves left = rem - RN(RN(rem/r)*r),
// which is 0 for rate 1 and at most 2^-52 * rem for rate sigma; with every
// duration below kFastHi = 2^22 ms that is < 1e-9, so each step finalizes at
// least one command and 3n steps drain a group (the fast path relies on it;
// the host selects it only for durations in [2^-60, 2^22)).  Beyond that a
// command may need a few more steps (rem shrinks by ~2^-52 per extra step),
// so the general path allows kSlowSteps steps per command.
constexpr double kFastHi = 0x1p22;
constexpr int kSlowSteps = 24;
constexpr int kMaxN = 16;         // 4-bit positions in a u64 sequence
constexpr int kStride = 16;       // doubles per kind row in shared memory

__device__ __forceinline__ int nib(uint64_t seq, int pos) {
    return (int)((seq >> (4 * pos)) & 0xFull);
}

template <bool FASTDIV>
__device__ __forceinline__ double divq(double x, double y, double ry) {
    if constexpr (FASTDIV) {
        double q0 = __dmul_rn(x, ry);
        double e = __fma_rn(-q0, y, x);
        return __fma_rn(e, ry, q0);
    } else {
        return __ddiv_rn(x, y);
    }
}

// Python's max(left, 0.0): the first argument unless 0.0 compares greater.
__device__ __forceinline__ double pymax0(double left) { return (0.0 > left) ? 0.0 : left; }

// Per-thread view of one task group's durations in shared memory.
struct Durs {
    const double* d;  // d[s*(k*kStride + t)], k = 0 HtD, 1 K, 2 DtH
    const double* r;  // 1/d, same layout
    int s = 1;        // 1: separate arrays; 2: interleaved {nd, 1/nd} pairs
    __device__ __forceinline__ double nd(int k, int t) const { return d[s * (k * kStride + t)]; }
    __device__ __forceinline__ double rc(int k, int t) const { return r[s * (k * kStride + t)]; }
};

// Optional full-timeline record (timeline mode only, general path).
struct TimelineOut {
    double* start;  // [n][3] by task index
    double* end;
};

// ---------------------------------------------------------------------------
// Simulator state.  DMA: 1 or 2 engines (engine.py:97-104).
// FAST: every stage of every task is non-null, so the three queues are the
// ordering itself and readiness reduces to head comparisons
//   K(p) ready  <=> HtD(p) finalized <=> p < headH        (engine.py:172-173)
//   DtH(p) ready <=> K(p) finalized  <=> p < headK        (:174-177)
// Otherwise (general) heads skip null stages (engine.py:129-151) and
// readiness uses per-kind done bitmasks over task ids.
// TRACK: also keep k_end and idle["K"] (heuristic.py:46, :74).
// ---------------------------------------------------------------------------
template <int DMA, bool FAST, bool FASTDIV, bool TRACK>
struct Sim {
    // inputs
    Durs D;
    uint64_t seq;
    int len;
    double sigma, rsig;
    // lanes: 2-DMA {0:HtD, 1:DtH, 2:K}; 1-DMA {0:XFER, 2:K}
    double now;
    double rem0, rem1, rem2;
    double nd0, nd1, nd2;
    double rc0, rc1, rc2;
    int h0, h1, h2;   // FAST: finalized count; general: head position/slot
    int kind0;        // 1-DMA: kind of the XFER head command (0 HtD / 2 DtH)
    bool run0, run1, run2;
    unsigned doneH, doneK, doneD;  // general path only
    unsigned nullH, nullK, nullD;
    int kfin;
    double kEnd, idleK;

    __device__ __forceinline__ void init(const Durs& d, uint64_t s, int n, double sg, double rsg,
                                         unsigned nH = 0, unsigned nK = 0, unsigned nD = 0) {
        D = d;
        seq = s;
        len = n;
        sigma = sg;
        rsig = rsg;
        now = 0.0;
        rem0 = rem1 = rem2 = 1.0;
        nd0 = nd1 = nd2 = 1.0;
        rc0 = rc1 = rc2 = 1.0;
        h0 = h1 = h2 = 0;
        kind0 = 0;
        run0 = run1 = run2 = false;
        kfin = 0;
        kEnd = 0.0;
        idleK = 0.0;
        if constexpr (!FAST) {
            nullH = nH;
            nullK = nK;
            nullD = nD;
            doneH = nH;
            doneK = nK;
            doneD = nD;
            if constexpr (DMA == 2) {
                h0 = skip(0, nullH);
                h1 = skip(0, nullD);
            } else {
                h0 = skipx(0);
            }
            h2 = skip(0, nullK);
        }
    }

    // next position >= p whose stage of the given null-mask is non-null
    __device__ __forceinline__ int skip(int p, unsigned nullmask) const {
        while (p < len && ((nullmask >> nib(seq, p)) & 1u)) ++p;
        return p;
    }
    // 1-DMA XFER queue slots: [HtD(p0..), DtH(p0..)] (engine.py:153-154)
    __device__ __forceinline__ int skipx(int s) const {
        while (s < 2 * len) {
            bool isH = s < len;
            int t = nib(seq, isH ? s : s - len);
            if (!(((isH ? nullH : nullD) >> t) & 1u)) break;
            ++s;
        }
        return s;
    }

    __device__ __forceinline__ bool drained() const {
        if constexpr (FAST) {
            if constexpr (DMA == 2) return h1 >= len;
            else return h0 >= 2 * len;
        } else {
            if constexpr (DMA == 2) return h0 >= len && h1 >= len && h2 >= len;
            else return h0 >= 2 * len && h2 >= len;
        }
    }

    __device__ __forceinline__ void startK(TimelineOut* tl) {
        int t = nib(seq, h2);
        nd2 = D.nd(1, t);
        rc2 = D.rc(1, t);
        rem2 = nd2;
        run2 = true;
        if constexpr (TRACK) {
            // idle_report (engine.py:68-80): K spans are FIFO == sorted
            if (kfin > 0 && now > kEnd) idleK = __dadd_rn(idleK, __dsub_rn(now, kEnd));
        }
        if (tl) tl->start[3 * t + 1] = now;
    }

    // One DeviceSim.step() (engine.py:182-232).  No-op once drained.
    __device__ __forceinline__ void step(TimelineOut* tl = nullptr) {
        const double INF = __longlong_as_double(0x7ff0000000000000ll);
        // ---- start phase (engine.py:188-194)
        if constexpr (DMA == 2) {
            if (!run0 && h0 < len) {
                int t = nib(seq, h0);
                nd0 = D.nd(0, t); rc0 = D.rc(0, t); rem0 = nd0; run0 = true;
                if (tl) tl->start[3 * t + 0] = now;
            }
            if constexpr (FAST) {
                if (!run2 && h2 < h0) startK(tl);
                if (!run1 && h1 < h2) {
                    int t = nib(seq, h1);
                    nd1 = D.nd(2, t); rc1 = D.rc(2, t); rem1 = nd1; run1 = true;
                }
            } else {
                if (!run2 && h2 < len && ((doneH >> nib(seq, h2)) & 1u)) startK(tl);
                if (!run1 && h1 < len) {
                    int t = nib(seq, h1);
                    if (((doneK & doneH) >> t) & 1u) {
                        nd1 = D.nd(2, t); rc1 = D.rc(2, t); rem1 = nd1; run1 = true;
                        if (tl) tl->start[3 * t + 2] = now;
                    }
                }
            }
        } else {
            if (!run0 && h0 < 2 * len) {
                bool isH = h0 < len;
                int t = nib(seq, isH ? h0 : h0 - len);
                bool ready;
                if constexpr (FAST) ready = isH || (h2 > h0 - len);
                else ready = isH || (((doneK & doneH) >> t) & 1u);
                if (ready) {
                    int k = isH ? 0 : 2;
                    kind0 = k;
                    nd0 = D.nd(k, t); rc0 = D.rc(k, t); rem0 = nd0; run0 = true;
                    if (tl) tl->start[3 * t + k] = now;
                }
            }
            if constexpr (FAST) {
                if (!run2 && h2 < len && h2 < h0) startK(tl);
            } else {
                if (!run2 && h2 < len && ((doneH >> nib(seq, h2)) & 1u)) startK(tl);
            }
        }
        const bool act = run0 | run1 | run2;
        // ---- rates (engine.py:200-208): both transfer directions slowed by
        // sigma while an HtD and a DtH execute together on a 2-DMA device
        bool ov = false;
        if constexpr (DMA == 2) ov = run0 && run1;
        // ---- dt (engine.py:210)
        double c0 = run0 ? (ov ? divq<FASTDIV>(rem0, sigma, rsig) : rem0) : INF;
        double c1 = INF;
        if constexpr (DMA == 2) c1 = run1 ? (ov ? divq<FASTDIV>(rem1, sigma, rsig) : rem1) : INF;
        double c2 = run2 ? rem2 : INF;
        double dt = fmin(fmin(c0, c1), c2);
        if (act) now = __dadd_rn(now, dt);  // engine.py:211
        // ---- remaining work (engine.py:212-214)
        const double dd = ov ? __dmul_rn(dt, sigma) : dt;
        rem0 = __dmul_rn(divq<FASTDIV>(pymax0(__dsub_rn(rem0, dd)), nd0, rc0), nd0);
        if constexpr (DMA == 2)
            rem1 = __dmul_rn(divq<FASTDIV>(pymax0(__dsub_rn(rem1, dd)), nd1, rc1), nd1);
        rem2 = __dmul_rn(divq<FASTDIV>(pymax0(__dsub_rn(rem2, dt)), nd2, rc2), nd2);
        // ---- finalize (engine.py:216-231); the order HtD, DtH, K only
        // orders the returned list, not the numbers
        const bool f0 = run0 && rem0 <= kEndEps;
        const bool f1 = (DMA == 2) && run1 && rem1 <= kEndEps;
        const bool f2 = run2 && rem2 <= kEndEps;
        if constexpr (FAST) {
            if (f0) { run0 = false; ++h0; }
            if (f1) { run1 = false; ++h1; }
            if (f2) { run2 = false; ++h2; }
            if (tl) {
                // FAST never runs with a timeline record
            }
        } else {
            if (f0) {
                run0 = false;
                if constexpr (DMA == 2) {
                    int t = nib(seq, h0);
                    doneH |= 1u << t;
                    if (tl) tl->end[3 * t + 0] = now;
                    h0 = skip(h0 + 1, nullH);
                } else {
                    bool isH = h0 < len;
                    int t = nib(seq, isH ? h0 : h0 - len);
                    if (isH) doneH |= 1u << t; else doneD |= 1u << t;
                    if (tl) tl->end[3 * t + (isH ? 0 : 2)] = now;
                    h0 = skipx(h0 + 1);
                }
            }
            if (f1) {
                int t = nib(seq, h1);
                run1 = false;
                doneD |= 1u << t;
                if (tl) tl->end[3 * t + 2] = now;
                h1 = skip(h1 + 1, nullD);
            }
            if (f2) {
                int t = nib(seq, h2);
                run2 = false;
                doneK |= 1u << t;
                if (tl) tl->end[3 * t + 1] = now;
                h2 = skip(h2 + 1, nullK);
            }
        }
        if constexpr (TRACK) {
            if (f2) { kEnd = now; ++kfin; }
        }
    }

    // DeviceSim.run (engine.py:237-241); returns false on a stall (cannot
    // happen without deps, kept as a guard).  Bound: see kSlowSteps.
    __device__ __forceinline__ bool run(TimelineOut* tl = nullptr) {
        const int max_steps = 3 * len * kSlowSteps;
        for (int s = 0; s < max_steps; ++s) {
            if (drained()) break;
            step(tl);
        }
        return drained();
    }
};

// ---------------------------------------------------------------------------
// FastSim: the all-stages-non-null path with the instruction count cut to
// the bone (the kernels are issue-bound, not FP64-bound).  Exactly the same
// arithmetic as Sim<FAST=true>; the differences are representational:
//  * idle lanes hold rem = 2^900 instead of a running flag in the dt min and
//    the update (no selects; 2^900 * (1/nd) cannot overflow for durations in
//    [2^-60, 2^22), and 2^900 - dt == 2^900);
//  * max(left, 0.0) (engine.py:214) is dropped: when left <= 0 the command
//    finalizes in this step with or without it (rw*nd <= 0 <= 1e-9), and a
//    finalized command's rw is never read again (engine.py:223);
//  * dt = min(rem_H/s, rem_D/s, rem_K) = min(RN(min(rem_H, rem_D)/s), rem_K):
//    RN(x/s) is monotone in x, so one division per step instead of two;
//  * {nd, 1/nd} of a (kind, task) is one predicated 16-byte shared load.
// Durations live in shared memory as double2 [3][16] at `base` (32-bit
// shared address): kind k, task t at base + k*256 + t*16.
// ---------------------------------------------------------------------------
constexpr double kBig = 0x1p900;
// a lane is idle iff its rem is the sentinel (>= 2^899): one integer compare
// on the high word instead of a running flag
constexpr int kIdleHi = 0x78200000;  // high word of 2^899

__device__ __forceinline__ bool idle(double r) { return __double2hiint(r) >= kIdleHi; }

// predicated {nd, 1/nd} load; on success rem = nd (a new command starts)
__device__ __forceinline__ void start_if(bool p, uint32_t addr, double& nd, double& rc, double& rem) {
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %4, 0;\n\t"
        "@q ld.shared.v2.f64 {%0, %1}, [%3];\n\t@q ld.shared.f64 %2, [%3];\n\t}"
        : "+d"(nd), "+d"(rc), "+d"(rem)
        : "r"(addr), "r"((int)p));
}
// the same with three 8-byte loads: no 16-byte register-pair alignment for
// {nd, 1/nd}, so under register pressure the compiler needs no predicated
// moves from a temporary quad (k_heuristic_fast: -6 instructions per step)
__device__ __forceinline__ void start_if_split(bool p, uint32_t addr, double& nd, double& rc, double& rem) {
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %4, 0;\n\t"
        "@q ld.shared.f64 %0, [%3];\n\t@q ld.shared.f64 %1, [%3+8];\n\t@q ld.shared.f64 %2, [%3];\n\t}"
        : "+d"(nd), "+d"(rc), "+d"(rem)
        : "r"(addr), "r"((int)p));
}
// LAYOUTs 2 and 3 of FastSim: nd and 1/nd in separate lane-interleaved
// arrays, 1/nd RCOFF bytes above nd
template <int RCOFF>
__device__ __forceinline__ void start_if_lanes(bool p, uint32_t addr, double& nd, double& rc, double& rem) {
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %4, 0;\n\t"
        "@q ld.shared.f64 %0, [%3];\n\t@q ld.shared.f64 %1, [%3+%5];\n\t@q ld.shared.f64 %2, [%3];\n\t}"
        : "+d"(nd), "+d"(rc), "+d"(rem)
        : "r"(addr), "r"((int)p), "n"(RCOFF));
}
__device__ __forceinline__ void mul_if(bool p, double& x, double y) {
    asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q mul.rn.f64 %0, %0, %1;\n\t}"
        : "+d"(x) : "d"(y), "r"((int)p));
}
__device__ __forceinline__ void add_if(bool p, double& x, double y) {
    asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q add.rn.f64 %0, %0, %1;\n\t}"
        : "+d"(x) : "d"(y), "r"((int)p));
}

__device__ __forceinline__ double dmin(double a, double b) { return (b < a) ? b : a; }

// idle sentinel by high word only (the low word is irrelevant: any value with
// that high word is ~2^900)
__device__ __forceinline__ double retire(double r) { return __hiloint2double(0x78300000, __double2loint(r)); }
// finalize of the lane that holds the group's last command: instead of the
// sentinel, the high word becomes 0 (rem ~ a subnormal), so later steps have
// dt ~ 0 and now + dt == now exactly -- a drained thread's steps are no-ops.
__device__ __forceinline__ double retire_or_drain(bool fin, double r, bool last) {
    const int hi = last ? 0 : 0x78300000;
    return __hiloint2double(fin ? hi : __double2hiint(r), __double2loint(r));
}

// byte offset (task*16) of the task at shift `sh` (= 4*position).  PRE: the
// sequence is stored pre-shifted left by 4 (positions 0..14 only).
template <bool PRE>
__device__ __forceinline__ uint32_t task_off(uint64_t seq, int sh) {
    if constexpr (PRE) return (uint32_t)(seq >> sh) & 0xF0u;
    else return ((uint32_t)(seq >> sh) & 0xFu) << 4;
}

// DEPS (2-DMA only): each task may wait for a prerequisite task to finish
// (engine.py:168-171, the NoReorder chains of workload.py:313-317); `dseq`
// holds, per position, 1 + the prerequisite's position (0: none), packed
// like `seq`.  With every stage non-null a task is finished exactly when its
// DtH finalized, and DtHs finalize in sequence order, so the gate is one
// extra condition on the HtD start: s1 >= 4 * (1 + prerequisite position).
#ifndef OSIM_LANE_MAD
#define OSIM_LANE_MAD 1
#endif
// LAYOUT of the durations in shared memory:
//  0: double2 {nd, 1/nd} rows [3][16] at `base` (kind k, task t at base + k*256 + t*16),
//     one 16-byte + one 8-byte load per command start;
//  1: the same rows, three 8-byte loads (start_if_split);
//  2: lane-interleaved arrays nd[48][32], rc[48][32] (one group per lane; kind
//     k, task t of lane l at base + (k*16 + t)*256 with base = array + 8*l,
//     1/nd 12288 bytes above): a warp's 8-byte loads of 32 different
//     (kind, task) entries are bank-conflict free;
//  3: the same with 16 groups per row (two lanes per group, l and l + 16):
//     task stride 128 bytes, 1/nd 6144 bytes above; each half-warp's 8-byte
//     loads touch 16 different groups, again conflict free.
template <int DMA, bool SIGP2, bool TRACK, bool PRE, bool DEPS = false, int LAYOUT = 0>
struct FastSim {
    static_assert(LAYOUT == 0 || LAYOUT == 4 || !PRE, "pre-shifted sequences assume the double2 rows");
    static constexpr int kDma = DMA;
    static constexpr bool kLanes = LAYOUT == 2 || LAYOUT == 3 || LAYOUT == 6;  // lane-interleaved arrays
    static constexpr bool kRegH = LAYOUT == 6;  // HtD durations from registers (set_htd), not shared memory
    static constexpr int kTSh = (LAYOUT == 3) ? 7 : 8;  // LAYOUTs 2/3/6: log2 bytes per task row
    static constexpr uint32_t KS = kLanes ? (16u << kTSh) : 256u;  // bytes per kind row
    static constexpr int kRcOff = (kRegH ? 32 : 48) << kTSh;  // LAYOUTs 2/3/6: 1/nd above nd
    static constexpr uint32_t KO_K = kRegH ? 0u : KS;       // kind row offsets (LAYOUT 6 stores K, DtH only)
    static constexpr uint32_t KO_D = kRegH ? KS : 2 * KS;
    // LAYOUTs 2/3/6: the task index (times the row stride in adr()); else the byte offset
    __device__ __forceinline__ static uint32_t toff(uint64_t sq, int sh) {
        if constexpr (kLanes) return (uint32_t)(sq >> sh) & 0xFu;
        else return task_off<PRE>(sq, sh);
    }
    // address of the (kind offset kofs, task offset t) entry; LAYOUT 4 (the
    // double2 rows at a 256-byte-aligned base held in a register): base | t
    // is one LOP3 with the task-offset mask and kofs folds into the load's
    // immediate -- no shared-window base rematerialized in the loops
    __device__ __forceinline__ uint32_t adr(uint32_t kofs, uint32_t t) const {
        if constexpr (LAYOUT == 4) return (base | t) + kofs;
        else if constexpr (kLanes) {
#if OSIM_LANE_MAD
            // one multiply-add for row * stride + base (the compiler otherwise
            // emits shift, mask and add for the masked-then-shifted index)
            uint32_t a;
            asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(a) : "r"(t), "n"(1 << kTSh), "r"(base));
            return a + kofs;
#else
            return base + kofs + (t << kTSh);
#endif
        } else return base + kofs + t;
    }
    // a command start: {nd, 1/nd} and rem = nd from shared memory
    __device__ __forceinline__ static void st_(bool p, uint32_t addr, double& nd, double& rc, double& rem) {
        if constexpr (LAYOUT == 1) start_if_split(p, addr, nd, rc, rem);
        else if constexpr (kLanes) start_if_lanes<kRcOff>(p, addr, nd, rc, rem);
        else start_if(p, addr, nd, rc, rem);
    }
    uint32_t base;
    double hnd, hrc, hnd2, hrc2;  // LAYOUT 6: {nd, 1/nd} of the next two HtDs to start (set_htd)
    uint64_t seq;   // packed ordering (pre-shifted by 4 when PRE)
    uint64_t dseq;  // DEPS: packed 1 + prerequisite position (pre-shifted like seq)
    int n4;         // 4*n
    double now;
    double r0, r1, r2;  // 2-DMA: HtD, DtH, K;  1-DMA: XFER, -, K.  kBig = idle
    double d0, d1, d2;
    double c0, c1, c2;
    int s0, s1, s2;     // 4 * finalized count per lane
    double kEnd, idleK;

    __device__ __forceinline__ void init(uint32_t b, uint64_t sq, int n) {
        base = b;
        seq = PRE ? (sq << 4) : sq;
        n4 = 4 * n;
        now = 0.0;
        r0 = r1 = r2 = kBig;
        d0 = d1 = d2 = 1.0;
        c0 = c1 = c2 = 1.0;
        s0 = s1 = s2 = 0;
        kEnd = 0.0;
        idleK = 0.0;
    }
    __device__ __forceinline__ void set_seq(uint64_t sq) { seq = pack_seq(sq); }
    // {nd, 1/nd} of the K and DtH heads (the running commands, if any) from
    // the duration rows: restoring a checkpoint that stores only the rems
    __device__ __forceinline__ void reload_kd() {
        ld_dc(adr(KO_D, toff(seq, s1)), d1, c1);
        ld_dc(adr(KO_K, toff(seq, s2)), d2, c2);
    }
    __device__ __forceinline__ static void ld_dc(uint32_t addr, double& nd, double& rc) {
        if constexpr (kLanes) {
            asm("ld.shared.f64 %0, [%2];\n\tld.shared.f64 %1, [%2+%3];" : "=d"(nd), "=d"(rc) : "r"(addr), "n"(kRcOff));
        } else {
            asm("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(nd), "=d"(rc) : "r"(addr));
        }
    }
    static constexpr bool kPre = PRE;
    __device__ __forceinline__ static uint64_t pack_seq(uint64_t sq) { return PRE ? (sq << 4) : sq; }
    // start the HtD at the queue head now (the HtD lane is idle and an HtD
    // is always ready): what the next step's start phase would do
    __device__ __forceinline__ void start_htd() {
        if constexpr (kRegH) reg_htd(true);
        else st_(true, adr(0, toff(seq, s0)), d0, c0, r0);
    }
    // LAYOUT 6: the durations of the next HtD the queue will start
    __device__ __forceinline__ void set_htd(double nd, double rc, double nd2 = 1.0, double rc2 = 1.0) {
        hnd = nd; hrc = rc; hnd2 = nd2; hrc2 = rc2;
    }
    __device__ __forceinline__ void reg_htd(bool st) {  // LAYOUT 6: start the pending HtD if st
        d0 = st ? hnd : d0; c0 = st ? hrc : c0; r0 = st ? hnd : r0;
        hnd = st ? hnd2 : hnd; hrc = st ? hrc2 : hrc;
    }
    __device__ __forceinline__ int finalized() const { return (s0 + s1 + s2) >> 2; }

    // checkpoint image (prefix sharing across calls, e.g. in shared memory)
    struct Ck {
        double now, r0, r1, r2, d0, d1, d2, c0, c1, c2, kEnd, idleK;
        int s0, s1, s2, pad;
    };
    __device__ __forceinline__ void save(Ck& k) const {
        k.now = now; k.r0 = r0; k.r1 = r1; k.r2 = r2; k.d0 = d0; k.d1 = d1; k.d2 = d2;
        k.c0 = c0; k.c1 = c1; k.c2 = c2; k.kEnd = kEnd; k.idleK = idleK;
        k.s0 = s0; k.s1 = s1; k.s2 = s2;
    }
    __device__ __forceinline__ void load(const Ck& k) {
        now = k.now; r0 = k.r0; r1 = k.r1; r2 = k.r2; d0 = k.d0; d1 = k.d1; d2 = k.d2;
        c0 = k.c0; c1 = k.c1; c2 = k.c2; kEnd = k.kEnd; idleK = k.idleK;
        s0 = k.s0; s1 = k.s1; s2 = k.s2;
    }
    // finalized HtD commands (the prefix-checkpoint test) for both modes
    __device__ __forceinline__ int htd_done() const { return s0 >> 2; }

    __device__ __forceinline__ bool drained() const {
        if constexpr (DMA == 2) return s1 >= n4;
        else return s0 >= 2 * n4;
    }

    __device__ __forceinline__ double upd(double rem, double dd, double nd, double rc) const {
        return __dmul_rn(divq<true>(__dsub_rn(rem, dd), nd, rc), nd);
    }

    // ---- phase-specialized steps (2-DMA).  Once every HtD has
    // finalized the HtD lane stays idle (rem = sentinel), so no transfer
    // overlap exists (rate 1 everywhere, engine.py:200-208) and step() reduces
    // exactly to step_kd(); once every K has finalized too it reduces to
    // step_d().  Same operations, same order, on the lanes that can run.
    __device__ __forceinline__ void step_kd() {
        static_assert(DMA == 2, "2-DMA only");
        const bool st2 = idle(r2) && s2 < n4;
        const bool st1 = idle(r1) && s1 < s2;
        k_idle_gap(st2);
        st_(st2, adr(KO_K, toff(seq, s2)), d2, c2, r2);
        st_(st1, adr(KO_D, toff(seq, s1)), d1, c1, r1);
        const double dt = dmin(r1, r2);
        now = __dadd_rn(now, dt);
        r2 = upd(r2, dt, d2, c2);
        r1 = upd(r1, dt, d1, c1);
        const bool f1 = r1 <= OSIM_FIN_EPS;
        r1 = retire_or_drain(f1, r1, s1 + 4 >= n4);
        s1 += f1 ? 4 : 0;
        if (r2 <= OSIM_FIN_EPS) {
            r2 = retire(r2);
            s2 += 4;
            if constexpr (TRACK) kEnd = now;
        }
    }
    __device__ __forceinline__ void step_d() {
        static_assert(DMA == 2, "2-DMA only");
        const bool st1 = idle(r1) && s1 < n4;
        st_(st1, adr(KO_D, toff(seq, s1)), d1, c1, r1);
        const double dt = r1;  // the only lane that can run (rem ~0 once drained)
        now = __dadd_rn(now, dt);
        r1 = upd(r1, dt, d1, c1);
        const bool f1 = r1 <= OSIM_FIN_EPS;
        r1 = retire_or_drain(f1, r1, s1 + 4 >= n4);
        s1 += f1 ? 4 : 0;
    }

    // ---- 1-DMA phase-specialized steps.  Once the XFER queue is past every
    // HtD (s0 >= n4) step() has isH false, and K(s2) is always ready
    // (s2 < n4 <= s0); once every K has finalized too the K lane stays idle
    // and only the XFER lane (the DtH block) runs.  Same operations, same
    // order, on the lanes that can run.
    __device__ __forceinline__ void step_1d() {
        static_assert(DMA == 1, "1-DMA only");
        const int ps = s0 - n4;
        const bool st0 = idle(r0) && s0 < 2 * n4 && s2 > ps;
        const bool st2 = idle(r2) && s2 < n4;
        k_idle_gap(st2);
        st_(st0, adr(KO_D, toff(seq, ps)), d0, c0, r0);
        st_(st2, adr(KO_K, toff(seq, s2)), d2, c2, r2);
        const double dt = dmin(r0, r2);
        now = __dadd_rn(now, dt);
        r0 = upd(r0, dt, d0, c0);
        r2 = upd(r2, dt, d2, c2);
        const bool f0 = r0 <= OSIM_FIN_EPS;
        r0 = retire_or_drain(f0, r0, s0 + 4 >= 2 * n4);
        s0 += f0 ? 4 : 0;
        if (r2 <= OSIM_FIN_EPS) {
            r2 = retire(r2);
            s2 += 4;
            if constexpr (TRACK) kEnd = now;
        }
    }
    // 1-DMA with the queue's last HtD already started (start_htd): the XFER
    // lane can only start DtHs (every HtD is finalized whenever it is idle), so
    // step() reduces to step_1d() plus the K readiness test on the HtD head
    __device__ __forceinline__ void step_1dk() {
        static_assert(DMA == 1, "1-DMA only");
        const int ps = s0 - n4;
        const bool st0 = idle(r0) && s0 < 2 * n4 && s2 > ps;
        const bool st2 = idle(r2) && s2 < n4 && s2 < s0;
        k_idle_gap(st2);
        st_(st0, adr(KO_D, toff(seq, ps)), d0, c0, r0);
        st_(st2, adr(KO_K, toff(seq, s2)), d2, c2, r2);
        const double dt = dmin(r0, r2);
        now = __dadd_rn(now, dt);
        r0 = upd(r0, dt, d0, c0);
        r2 = upd(r2, dt, d2, c2);
        const bool f0 = r0 <= OSIM_FIN_EPS;
        r0 = retire_or_drain(f0, r0, s0 + 4 >= 2 * n4);
        s0 += f0 ? 4 : 0;
        if (r2 <= OSIM_FIN_EPS) {
            r2 = retire(r2);
            s2 += 4;
            if constexpr (TRACK) kEnd = now;
        }
    }
    __device__ __forceinline__ void step_1dd() {
        static_assert(DMA == 1, "1-DMA only");
        const bool st0 = idle(r0) && s0 < 2 * n4;
        st_(st0, adr(KO_D, toff(seq, s0 - n4)), d0, c0, r0);
        const double dt = r0;  // the only lane that can run (rem ~0 once drained)
        now = __dadd_rn(now, dt);
        r0 = upd(r0, dt, d0, c0);
        const bool f0 = r0 <= OSIM_FIN_EPS;
        r0 = retire_or_drain(f0, r0, s0 + 4 >= 2 * n4);
        s0 += f0 ? 4 : 0;
    }

    // run_phased (2-DMA) that also calls snap(steps so far) right after the
    // step in which this lane's HtD count reaches `target` (the state a
    // lock-step advance_to(target) would stop at)
    template <int PHF, class F>
    __device__ __forceinline__ void run_phased_snap(int rest, double sigma, double rsig, int target, F&& snap) {
        constexpr int kF = DMA == 2 ? PHF : 2;  // full steps per vote
        int st = 0;
        bool got = false;
#pragma unroll 1
        for (; st < rest; st += kF) {
            if (__all_sync(0xffffffffu, s0 >= n4)) break;
#pragma unroll
            for (int r = 0; r < kF; ++r) {
                step<true>(sigma, rsig);
                if (!got && (s0 >> 2) == target) {
                    got = true;
                    snap(st + r + 1);
                }
            }
        }
        if constexpr (DMA == 2) {
#pragma unroll 1
            for (; st < rest; st += OSIM_PH_KD) {
                if (__all_sync(0xffffffffu, s2 >= n4)) break;
#pragma unroll
                for (int r = 0; r < OSIM_PH_KD; ++r) step_kd();
            }
#pragma unroll 2
            for (; st < rest; ++st) step_d();
        } else {
#pragma unroll 1
            for (; st < rest; st += 2) {
                if (__all_sync(0xffffffffu, s2 >= n4)) break;
                step_1d();
                step_1d();
            }
#pragma unroll 2
            for (; st < rest; ++st) step_1dd();
        }
    }

    // `rest` steps in warp lock-step, switching to the specialized steps as
    // soon as the whole warp has drained its HtD (then K) lanes
    // H0 = false: see step(); the heuristic's candidate replays start the
    // candidate's HtD (the queue's last) before the first step
    template <bool H0 = true, int PHF = OSIM_PH_FULL>
    __device__ __forceinline__ void run_phased(int rest, double sigma, double rsig) {
        int st = 0;
        if constexpr (DMA == 2) {
#pragma unroll 1
            for (; st < rest; st += PHF) {
                if (__all_sync(0xffffffffu, s0 >= n4)) break;
#pragma unroll
                for (int r = 0; r < PHF; ++r) step<H0>(sigma, rsig);
            }
#pragma unroll 1
            for (; st < rest; st += OSIM_PH_KD) {
                if (__all_sync(0xffffffffu, s2 >= n4)) break;
#pragma unroll
                for (int r = 0; r < OSIM_PH_KD; ++r) step_kd();
            }
#pragma unroll 2
            for (; st < rest; ++st) step_d();
        } else if constexpr (H0) {
#pragma unroll 1
            for (; st < rest; st += 2) {
                if (__all_sync(0xffffffffu, s0 >= n4)) break;
                step(sigma, rsig);
                step(sigma, rsig);
            }
#pragma unroll 1
            for (; st < rest; st += 2) {
                if (__all_sync(0xffffffffu, s2 >= n4)) break;
                step_1d();
                step_1d();
            }
#pragma unroll 2
            for (; st < rest; ++st) step_1dd();
        } else {  // the last HtD already started: K+XFER-DtH steps, then XFER only
#pragma unroll 1
            for (; st < rest; st += 2) {
                if (__all_sync(0xffffffffu, s2 >= n4)) break;
                step_1dk();
                step_1dk();
            }
#pragma unroll 2
            for (; st < rest; ++st) step_1dd();
        }
    }

    __device__ __forceinline__ void k_idle_gap(bool st2) {
        if constexpr (TRACK) {
            // idle_report (engine.py:68-80) over K spans in FIFO (= sorted) order
            const double gap = __dsub_rn(now, kEnd);
            add_if(st2 && s2 > 0 && now > kEnd, idleK, gap);
        }
    }

    // H0 = false (2-DMA): the caller has already started the last HtD of the
    // queue, so no HtD can start in this step and its test and load are
    // skipped (st0 would be false)
    template <bool H0 = true>
    __device__ __forceinline__ void step(double sigma, double rsig) {
        // ---- start phase (engine.py:188-194); readiness in the all-non-null
        // case: K(p) needs HtD(p) finalized, DtH(p) needs K(p) finalized
        if constexpr (DMA == 2) {
            bool st0 = H0 && idle(r0) && s0 < n4;
            if constexpr (DEPS) st0 = st0 && s1 >= (int)(task_off<PRE>(dseq, s0) >> 2);
            const bool st2 = idle(r2) && s2 < s0;
            const bool st1 = idle(r1) && s1 < s2;
            k_idle_gap(st2);
            if constexpr (H0) {
                if constexpr (kRegH) {  // the pending HtD's durations (set_htd)
                    reg_htd(st0);
                } else {
                    st_(st0, adr(0, toff(seq, s0)), d0, c0, r0);
                }
            }
            st_(st2, adr(KO_K, toff(seq, s2)), d2, c2, r2);
            st_(st1, adr(KO_D, toff(seq, s1)), d1, c1, r1);
        } else {
            const bool isH = s0 < n4;
            const int ps = isH ? s0 : s0 - n4;
            const bool st0 = idle(r0) && s0 < 2 * n4 && (isH || s2 > ps);
            const bool st2 = idle(r2) && s2 < n4 && s2 < s0;
            k_idle_gap(st2);
            if constexpr (kRegH) {  // an XFER HtD from the pending registers, a DtH from shared memory
                st_(st0 && !isH, adr(KO_D, toff(seq, ps)), d0, c0, r0);
                reg_htd(st0 && isH);
            } else {
                st_(st0, adr(isH ? 0u : 2 * KS, toff(seq, ps)), d0, c0, r0);
            }
            st_(st2, adr(KO_K, toff(seq, s2)), d2, c2, r2);
        }
        // ---- dt (engine.py:200-210)
        double dt, dd;
        if constexpr (DMA == 2) {
            const bool ov = !idle(r0) && !idle(r1);
            double m = dmin(r0, r1);
            if constexpr (SIGP2) {
#if OSIM_EXPSHIFT
                // sigma = 2^-e: with both transfers running (ov) m = min of two
                // running commands' rem, a normal double in [2^-60, 2^22] (a
                // command starts with rem = nd >= 2^-60 and finalizes once rem
                // <= 1e-9), so m / sigma is m with e added to its exponent, and
                // dt * sigma (dt = min(m / sigma, rem_K) >= 2^-60) is dt with e
                // subtracted: exact, and one integer add on the high word each
                // instead of a select, a zeroed low word and a multiply.  Without
                // ov the factors are 1.0 (unchanged values; drained or idle
                // lanes' sentinels never get shifted).
                const int sh = ov ? __double2hiint(rsig) - 0x3FF00000 : 0;
                m = __hiloint2double(__double2hiint(m) + sh, __double2loint(m));
                dt = dmin(m, r2);
                dd = __hiloint2double(__double2hiint(dt) - sh, __double2loint(dt));
#else
                // sigma, 1/sigma and 1.0 are powers of two (low word 0): select
                // the factor's high word and multiply unconditionally
                // (x * 1.0 == x exactly), one integer select instead of a
                // 64-bit select of the product
                m = __dmul_rn(m, __hiloint2double(ov ? __double2hiint(rsig) : 0x3FF00000, 0));
                dt = dmin(m, r2);
                dd = __dmul_rn(dt, __hiloint2double(ov ? __double2hiint(sigma) : 0x3FF00000, 0));
#endif
            } else {
                if (ov) m = divq<true>(m, sigma, rsig);
                dt = dmin(m, r2);
                dd = dt;
                mul_if(ov, dd, sigma);
            }
        } else {
            dt = dmin(r0, r2);
            dd = dt;
        }
        now = __dadd_rn(now, dt);  // engine.py:211
        // ---- update + finalize (engine.py:212-231).  A finalized lane goes
        // idle by setting only the high word of rem to the sentinel's.  The
        // command that drains the group (the last DtH: 2-DMA lane 1, 1-DMA
        // lane 0) instead leaves rem = 0, so every later step has dt = 0 and
        // is a no-op (drained threads keep stepping in warp lock-step).
        r0 = upd(r0, dd, d0, c0);
        r2 = upd(r2, dt, d2, c2);
        if constexpr (DMA == 2) r1 = upd(r1, dd, d1, c1);
        if constexpr (DMA == 2) {
            if (r0 <= OSIM_FIN_EPS) { r0 = retire(r0); s0 += 4; }
            const bool f1 = r1 <= OSIM_FIN_EPS;
            r1 = retire_or_drain(f1, r1, s1 + 4 >= n4);
            s1 += f1 ? 4 : 0;
        } else {
            const bool f0 = r0 <= OSIM_FIN_EPS;
            r0 = retire_or_drain(f0, r0, s0 + 4 >= 2 * n4);
            s0 += f0 ? 4 : 0;
        }
        if (r2 <= OSIM_FIN_EPS) {
            r2 = retire(r2);
            s2 += 4;
            if constexpr (TRACK) kEnd = now;
        }
    }
};

// FastSim generalized to null stages (see osim_null.cuh for the contract):
// position heads, find-first-set skipping over per-sequence null masks,
// "head passed or stage null" readiness, dt clamped to 0 once all lanes idle.
template <int DMA, bool SIGP2, bool TRACK = false>
struct NullSim {
    uint32_t base;
    uint64_t seq;
    int n, n4;
    unsigned mH, mK, mX;  // position null masks (HtD, K; mX: 1-DMA XFER slots, 2-DMA DtH)
    double now;
    double r0, r1, r2, d0, d1, d2, c0, c1, c2;
    int s0, s1, s2;  // 4 * head position: HtD (1-DMA: XFER slot), DtH, K
    double kEnd, idleK;  // TRACK: last K end, idle_report's K gaps (engine.py:68-80)
    bool kfin;           // TRACK: some K has finalized

    // next non-null slot after s (4x units) in mask m over `lim` slots
    __device__ __forceinline__ static int next(unsigned m, int s, int lim) {
        const int p = s >> 2;
        const unsigned above = p >= 31 ? 0u : (~0u << (p + 1));
        const unsigned in = lim >= 32 ? ~0u : ((1u << lim) - 1u);
        const unsigned c = ~m & above & in;
        return 4 * (c ? __ffs(c) - 1 : lim);
    }
    __device__ __forceinline__ static int first(unsigned m, int lim) {
        const unsigned in = lim >= 32 ? ~0u : ((1u << lim) - 1u);
        const unsigned c = ~m & in;
        return 4 * (c ? __ffs(c) - 1 : lim);
    }
    __device__ __forceinline__ bool nul(unsigned m, int s) const { return (m >> (s >> 2)) & 1u; }

    // tH/tK/tD: null-stage masks by task id
    __device__ __forceinline__ void init(uint32_t b, uint64_t sq, int nn, unsigned tH, unsigned tK, unsigned tD) {
        base = b;
        seq = sq;
        n = nn;
        n4 = 4 * nn;
        unsigned pH = 0, pK = 0, pD = 0;
        for (int p = 0; p < nn; ++p) {
            const int t = nib(sq, p);
            pH |= ((tH >> t) & 1u) << p;
            pK |= ((tK >> t) & 1u) << p;
            pD |= ((tD >> t) & 1u) << p;
        }
        mH = pH;
        mK = pK;
        now = 0.0;
        r0 = r1 = r2 = kBig;
        d0 = d1 = d2 = c0 = c1 = c2 = 1.0;
        kEnd = 0.0;
        idleK = 0.0;
        kfin = false;
        s2 = first(pK, nn);
        if constexpr (DMA == 2) {
            mX = pD;
            s0 = first(pH, nn);
            s1 = first(pD, nn);
        } else {
            mX = pH | (pD << nn);
            s0 = first(mX, 2 * nn);
            s1 = 0;
        }
    }

    __device__ __forceinline__ bool drained() const {
        if constexpr (DMA == 2) return s0 >= n4 && s1 >= n4 && s2 >= n4 && idle(r0) && idle(r1) && idle(r2);
        else return s0 >= 2 * n4 && s2 >= n4 && idle(r0) && idle(r2);
    }

    __device__ __forceinline__ double upd(double rem, double dd, double nd, double rc) const {
        return __dmul_rn(divq<true>(__dsub_rn(rem, dd), nd, rc), nd);
    }

    __device__ __forceinline__ void step(double sigma, double rsig) {
        // ---- start phase (engine.py:188-194)
        if constexpr (DMA == 2) {
            const bool st0 = idle(r0) && s0 < n4;
            const bool st2 = idle(r2) && s2 < n4 && (s2 < s0 || nul(mH, s2));
            const bool st1 = idle(r1) && s1 < n4 && (s1 < s2 || nul(mK, s1)) && (s1 < s0 || nul(mH, s1));
            k_idle_gap(st2);
            start_if(st0, base + task_off<false>(seq, s0), d0, c0, r0);
            start_if(st2, base + 256 + task_off<false>(seq, s2), d2, c2, r2);
            start_if(st1, base + 512 + task_off<false>(seq, s1), d1, c1, r1);
        } else {
            const bool isH = s0 < n4;
            const int ps = isH ? s0 : s0 - n4;
            const bool st0 = idle(r0) && s0 < 2 * n4 && (isH || ps < s2 || nul(mK, ps));
            const bool st2 = idle(r2) && s2 < n4 && (s2 < s0 || nul(mH, s2));
            k_idle_gap(st2);
            start_if(st0, base + (isH ? 0u : 512u) + task_off<false>(seq, ps), d0, c0, r0);
            start_if(st2, base + 256 + task_off<false>(seq, s2), d2, c2, r2);
        }
        // ---- dt (engine.py:200-210); every lane idle (drained): dt = 0
        double dt, dd;
        if constexpr (DMA == 2) {
            const bool ov = !idle(r0) && !idle(r1);
            double m = dmin(r0, r1);
            if constexpr (SIGP2) {
#if OSIM_EXPSHIFT
                // as FastSim::step: exponent shifts of running commands' rems (ov)
                const int sh = ov ? __double2hiint(rsig) - 0x3FF00000 : 0;
                m = __hiloint2double(__double2hiint(m) + sh, __double2loint(m));
                dt = dmin(m, r2);
                dd = __hiloint2double(__double2hiint(dt) - sh, __double2loint(dt));
#else
                m = __dmul_rn(m, __hiloint2double(ov ? __double2hiint(rsig) : 0x3FF00000, 0));
                dt = dmin(m, r2);
                dd = __dmul_rn(dt, __hiloint2double(ov ? __double2hiint(sigma) : 0x3FF00000, 0));
#endif
            } else {
                if (ov) m = divq<true>(m, sigma, rsig);
                dt = dmin(m, r2);
                dd = dt;
                mul_if(ov, dd, sigma);
            }
        } else {
            dt = dmin(r0, r2);
            dd = dt;
        }
        if (idle(dt)) { dt = 0.0; dd = 0.0; }
        now = __dadd_rn(now, dt);  // engine.py:211
        // ---- update + finalize (engine.py:212-231)
        r0 = upd(r0, dd, d0, c0);
        r2 = upd(r2, dt, d2, c2);
        if constexpr (DMA == 2) r1 = upd(r1, dd, d1, c1);
        if (r0 <= kEndEps) {
            r0 = retire(r0);
            if constexpr (DMA == 2) s0 = next(mH, s0, n);
            else s0 = next(mX, s0, 2 * n);
        }
        if constexpr (DMA == 2) {
            if (r1 <= kEndEps) { r1 = retire(r1); s1 = next(mX, s1, n); }
        }
        if (r2 <= kEndEps) {
            r2 = retire(r2);
            s2 = next(mK, s2, n);
            if constexpr (TRACK) {
                kEnd = now;
                kfin = true;
            }
        }
    }

    // idle_report over K spans in FIFO (= sorted) order, as FastSim
    __device__ __forceinline__ void k_idle_gap(bool st2) {
        if constexpr (TRACK) {
            const double gap = __dsub_rn(now, kEnd);
            add_if(st2 && kfin && now > kEnd, idleK, gap);
        }
    }
};

// Lexicographic unrank of `r` into a packed sequence (itertools.permutations
// order == Lehmer rank order, oracle.py:125).
template <int N>
__device__ __forceinline__ uint64_t unrank(uint64_t r) {
    uint64_t avail = 0xFEDCBA9876543210ull;
    uint64_t seq = 0;
    if constexpr (N <= 12) {
        uint32_t rr = (uint32_t)r;
#pragma unroll
        for (int i = 0; i < N; ++i) {
            constexpr uint32_t dummy = 0;
            (void)dummy;
            uint32_t f = 1;
#pragma unroll
            for (int j = 2; j <= N - 1 - i; ++j) f *= (uint32_t)j;
            uint32_t d = rr / f;
            rr -= d * f;
            uint64_t t = (avail >> (4 * d)) & 0xFull;
            seq |= t << (4 * i);
            uint64_t low = (1ull << (4 * d)) - 1ull;
            avail = (avail & low) | ((avail >> 4) & ~low);
        }
    } else {
#pragma unroll
        for (int i = 0; i < N; ++i) {
            uint64_t f = 1;
#pragma unroll
            for (int j = 2; j <= N - 1 - i; ++j) f *= (uint64_t)j;
            uint64_t d = r / f;
            r -= d * f;
            uint64_t t = (avail >> (4 * d)) & 0xFull;
            seq |= t << (4 * i);
            uint64_t low = (1ull << (4 * d)) - 1ull;
            avail = (avail & low) | ((avail >> 4) & ~low);
        }
    }
    return seq;
}

// Runtime-n unrank (general path).
__device__ __forceinline__ uint64_t unrank_rt(uint64_t r, int n) {
    uint64_t avail = 0xFEDCBA9876543210ull;
    uint64_t seq = 0;
    for (int i = 0; i < n; ++i) {
        uint64_t f = 1;
        for (int j = 2; j <= n - 1 - i; ++j) f *= (uint64_t)j;
        uint64_t d = r / f;
        r -= d * f;
        uint64_t t = (avail >> (4 * d)) & 0xFull;
        seq |= t << (4 * i);
        uint64_t low = (1ull << (4 * d)) - 1ull;
        avail = (avail & low) | ((avail >> 4) & ~low);
    }
    return seq;
}

// CPython builtin sum() over doubles (bltinmodule.c builtin_sum_impl):
// 3.12+ Neumaier compensation, <=3.11 naive; the int start 0 is added first.
struct PySum {
    double f, c;
    bool any;
    __device__ __forceinline__ void reset() { f = 0.0; c = 0.0; any = false; }
    __device__ __forceinline__ void add(double x, int mode) {
        if (!any) { f = __dadd_rn(0.0, x); any = true; return; }
        if (mode) {
            double t = __dadd_rn(f, x);
            if (fabs(f) >= fabs(x)) c = __dadd_rn(c, __dadd_rn(__dsub_rn(f, t), x));
            else c = __dadd_rn(c, __dadd_rn(__dsub_rn(x, t), f));
            f = t;
        } else {
            f = __dadd_rn(f, x);
        }
    }
    __device__ __forceinline__ double result(int mode) const {
        if (mode && c != 0.0 && isfinite(c)) return __dadd_rn(f, c);
        return f;
    }
};

}  // namespace osim
