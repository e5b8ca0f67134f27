// osim_capi.cu -- the extern "C" boundary (include/offsim_b200.h): argument
// validation with the reference's error semantics, device/stream/scratch
// management, kernel dispatch and multi-device sharding.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <mutex>
#include <thread>
#include <string>
#include <array>
#include <vector>

#include "osim_deps.cuh"
#include "osim_launch.cuh"
#include "osim_micro.cuh"
#include "osim_harness.cuh"
#include "osim_null.cuh"

using namespace osim;

namespace {

thread_local std::string g_err;
thread_local int g_thread_dev = -1;

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CK(call)                                                                          \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess)                                                            \
            return fail(OSIM_ECUDA, "%s failed: %s", #call, cudaGetErrorString(e_));      \
    } while (0)

struct DevCtx {
    int dev = 0;
    int sms = 148;
    cudaStream_t stream = nullptr;
    cudaStream_t stream2 = nullptr;  // second copy/compute stream for pipelined host calls
    cudaEvent_t ev = nullptr;
    void* scratch = nullptr;
    size_t scratch_bytes = 0;
    int* d_err = nullptr;
    unsigned* d_done = nullptr;  // last-CTA counter of the fused final reductions (kept at 0)
    AuxBuf aux[2];               // launchers' temporaries, per stream (stream, stream2)
    std::mutex mu;
};

std::mutex g_init_mu;
std::vector<DevCtx*> g_devs;

int ensure_init() {
    std::lock_guard<std::mutex> lk(g_init_mu);
    if (!g_devs.empty()) return 0;
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count <= 0)
        return fail(OSIM_ENODEV, "no CUDA device available (%s)", cudaGetErrorString(e));
    // OSIM_VIRTUAL_DEVICES=<k> (testing only): k library devices, device i on
    // physical GPU i % count, each with its own streams, scratch, error flag
    // and lock -- so the n_dev > 1 host paths (sharding, per-device
    // validation, host-side merges) run, and are tested, on a one-GPU box
    int nctx = count;
    if (const char* e = std::getenv("OSIM_VIRTUAL_DEVICES")) {
        const int k = std::atoi(e);
        if (k > count && k <= 64) nctx = k;
    }
    for (int i = 0; i < nctx; ++i) {
        const int d = i % count;
        DevCtx* c = new DevCtx();
        c->dev = d;
        CK(cudaSetDevice(d));
        CK(cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, d));
        CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&c->stream2, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&c->ev, cudaEventDisableTiming));
        CK(cudaMalloc(&c->d_err, sizeof(int)));
        CK(cudaMemset(c->d_err, 0, sizeof(int)));
        CK(cudaMalloc(&c->d_done, sizeof(unsigned)));
        CK(cudaMemset(c->d_done, 0, sizeof(unsigned)));
        g_devs.push_back(c);
    }
    return 0;
}

int cur_dev() {
    if (g_thread_dev >= 0) return g_thread_dev;
    int d = 0;
    cudaGetDevice(&d);
    return d < (int)g_devs.size() ? d : 0;
}

// grow-only per-device scratch; caller holds c->mu
int scratch(DevCtx* c, size_t bytes, void** p) {
    if (bytes > c->scratch_bytes) {
        if (c->scratch) cudaFree(c->scratch);
        c->scratch = nullptr;
        size_t want = bytes < (1u << 20) ? (1u << 20) : bytes + bytes / 4;
        CK(cudaMalloc(&c->scratch, want));
        c->scratch_bytes = want;
    }
    *p = c->scratch;
    return 0;
}

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

// Give back a scratch buffer that one call grew past `keep` bytes (the exact
// median of a 13-task space holds 56 GB of makespans): later calls
// re-allocate what they need.  8 GB keeps the 12-task space's (3.8 GB of
// makespans + compaction, 5.4 GB with the 25 % headroom) resident between
// calls: re-allocating it cost ~7 ms per call.  Caller holds c->mu; the
// device is idle.
void trim_scratch(DevCtx* c, size_t keep = size_t(8) << 30) {
    if (c->scratch && c->scratch_bytes > keep) {
        cudaFree(c->scratch);
        c->scratch = nullptr;
        c->scratch_bytes = 0;
    }
}

// ---- validation (model.py:63-71, 91-100; engine.py:129-130, 258-259) -----
int check_common(int n, int dma, double sigma, int maxn = kMaxN) {
    if (n < 1) return fail(OSIM_EINVAL, "task group must be non-empty");
    if (n > maxn) return fail(OSIM_EINVAL, "n=%d exceeds the supported maximum of %d tasks", n, maxn);
    if (dma != 1 && dma != 2) return fail(OSIM_EINVAL, "dma_engines must be 1 or 2, got %d", dma);
    if (!(sigma > 0.0 && sigma <= 1.0)) return fail(OSIM_EINVAL, "overlap_sigma must be in (0, 1]");
    return 0;
}

// One pass over the durations: the reference's validity rules
// (model.py:95-100, engine.py:129-130) and fast-path eligibility (every
// stage non-null and in [2^-60, 2^22)); split over host threads for large
// batches.  Reports the lowest offending task, as a serial scan would.
struct ScanPart {
    uint64_t bad = ~0ull;
    int why = 0;  // 1 = negative / non-finite, 2 = no commands
    bool fast = true;   // every stage in the FastSim range
    bool nfast = true;  // every stage 0 or in the FastSim range (NullSim)
};

void scan_range(const double* d, uint64_t t0, uint64_t t1, ScanPart& r) {
    const double lo = 0x1p-60, hi = 0x1p22;  // see kFastHi (osim_sim.cuh)
    bool fast = true, nfast = true;
    for (uint64_t t = t0; t < t1; ++t) {
        const double h = d[3 * t], k = d[3 * t + 1], x = d[3 * t + 2];
        if (!(h >= 0.0 && k >= 0.0 && x >= 0.0 && h <= 1.7976931348623157e308 && k <= 1.7976931348623157e308 &&
              x <= 1.7976931348623157e308)) {
            r.bad = t; r.why = 1; break;
        }
        if (h <= 0 && k <= 0 && x <= 0) { r.bad = t; r.why = 2; break; }
        fast = fast && h >= lo && h < hi && k >= lo && k < hi && x >= lo && x < hi;
        nfast = nfast && (h == 0.0 || (h >= lo && h < hi)) && (k == 0.0 || (k >= lo && k < hi)) &&
                (x == 0.0 || (x >= lo && x < hi));
    }
    r.fast = fast;
    r.nfast = nfast;
}

int scan_durs(const double* durs, uint64_t tasks, double sigma, int* fast) {
    if (!durs) return fail(OSIM_EINVAL, "durations pointer is NULL");
    unsigned nt = tasks >= (1ull << 18) ? std::thread::hardware_concurrency() : 1u;
    if (nt < 1) nt = 1;
    if (nt > 32) nt = 32;
    std::vector<ScanPart> parts(nt);
    if (nt == 1) {
        scan_range(durs, 0, tasks, parts[0]);
    } else {
        std::vector<std::thread> th;
        for (unsigned i = 0; i < nt; ++i)
            th.emplace_back(scan_range, durs, tasks * i / nt, tasks * (i + 1) / nt, std::ref(parts[i]));
        for (auto& t : th) t.join();
    }
    bool f = sigma >= 0x1p-60, nf = f;
    for (const ScanPart& p : parts) {
        if (p.bad != ~0ull) {
            if (p.why == 1)
                return fail(OSIM_EINVAL, "task %llu: durations must be finite and non-negative",
                            (unsigned long long)p.bad);
            return fail(OSIM_EINVAL, "task %llu has no commands", (unsigned long long)p.bad);
        }
        f = f && p.fast;
        nf = nf && p.nfast;
    }
    // 1: FastSim path; 2: null stages in the fast range (NullSim); 0: general
    if (fast) *fast = f ? 1 : (nf ? 2 : 0);
    return 0;
}

int check_durs(const double* durs, uint64_t tasks) { return scan_durs(durs, tasks, 1.0, nullptr); }

// micro_simulate resolves stage times without DeviceSim.submit's checks
// (oracle.py:72-76): a task without commands is allowed (it has no queue
// entries); durations must still be finite and non-negative
int check_durs_micro(const double* durs, uint64_t tasks) {
    if (!durs) return fail(OSIM_EINVAL, "durations pointer is NULL");
    for (uint64_t i = 0; i < 3 * tasks; ++i)
        if (!(durs[i] >= 0.0 && durs[i] < HUGE_VAL))
            return fail(OSIM_EINVAL, "task %llu: durations must be finite and non-negative",
                        (unsigned long long)(i / 3));
    return 0;
}

// each row of id ranks must be a permutation of range(n) (unique ids)
int check_id_ranks(const uint8_t* id_rank, uint64_t B, int n) {
    unsigned nt = B >= (1ull << 16) ? std::thread::hardware_concurrency() : 1u;
    if (nt < 1) nt = 1;
    if (nt > 32) nt = 32;
    std::vector<uint64_t> bad(nt, ~0ull);
    auto work = [&](unsigned i) {
        for (uint64_t b = B * i / nt; b < B * (i + 1) / nt; ++b) {
            uint64_t seen = 0;
            for (int j = 0; j < n; ++j) {
                const unsigned v = id_rank[b * n + j];
                if (v >= (unsigned)n || ((seen >> v) & 1ull)) { bad[i] = b; return; }
                seen |= 1ull << v;
            }
        }
    };
    if (nt == 1) work(0);
    else {
        std::vector<std::thread> th;
        for (unsigned i = 0; i < nt; ++i) th.emplace_back(work, i);
        for (auto& t : th) t.join();
    }
    for (uint64_t b : bad)
        if (b != ~0ull)
            return fail(OSIM_EINVAL, "group %llu: id ranks must be a permutation (duplicate task id?)",
                        (unsigned long long)b);
    return 0;
}

uint64_t factorial(int n) {
    uint64_t f = 1;
    for (int i = 2; i <= n; ++i) f *= (uint64_t)i;
    return f;
}

template <class K>
int grid_for(K kernel, int threads, size_t smem, const DevCtx* c, uint64_t work_blocks) {
    return osim::grid_for_sms(kernel, threads, smem, c->sms, work_blocks);
}

// NoReorder prefix-sharing run length (ranks per thread); OSIM_F1_RUN
// overrides it for tuning (tools/f1_speed.py)
int f1_run_len() {
    static const int v = [] {
        const char* e = std::getenv("OSIM_F1_RUN");
        const int x = e ? std::atoi(e) : 0;
        return (x >= 1 && x <= 4096) ? x : 32;
    }();
    return v;
}

bool sigma_pow2(double sigma) {
    int e;
    double m = std::frexp(sigma, &e);
    return m == 0.5 && e > -900;
}

int launch_exh_fast_dispatch(int dma, int n, DevCtx* c, cudaStream_t st, const double* d_durs, double sigma,
                             uint64_t lo, uint64_t hi, double thr, Part* parts, int max_parts, double* d_ms,
                             int* g, osim_summary* d_out, unsigned long long* d_below, unsigned shard = 0,
                             unsigned shards = 1) {
    const LaunchCfg cfg{c->sms, st};
    const int L = pfx_l_for(n);
    unsigned* dn = c->d_done;
    int rc;
    if (dma == 2)
        rc = sigma_pow2(sigma)
                 ? exh_fast_launch_d2s1(n, L, cfg, d_durs, sigma, lo, hi, thr, parts, max_parts, d_ms, g, d_out,
                                        d_below, dn, shard, shards)
                 : exh_fast_launch_d2s0(n, L, cfg, d_durs, sigma, lo, hi, thr, parts, max_parts, d_ms, g, d_out,
                                        d_below, dn, shard, shards);
    else
        rc = exh_fast_launch_d1(n, L, cfg, d_durs, sigma, lo, hi, thr, parts, max_parts, d_ms, g, d_out, d_below,
                                dn, shard, shards);
    if (rc) return fail(OSIM_EINVAL, "unsupported n=%d", n);
    return 0;
}

int launch_batch_fast_dispatch(int dma, int n, DevCtx* c, cudaStream_t st, const double* d_durs, uint64_t B,
                               double sigma, osim_summary* d_out) {
    const LaunchCfg cfg{c->sms, st};
    const int L = pfx_l_for(n);
    int rc = dma == 2 ? batch_fast_launch_d2(n, L, sigma_pow2(sigma), cfg, d_durs, B, sigma, d_out)
                      : batch_fast_launch_d1(n, L, cfg, d_durs, B, sigma, d_out);
    if (rc) return fail(OSIM_EINVAL, "unsupported n=%d", n);
    return 0;
}

// Enqueue exhaustive over [lo, hi) and its final reduce into d_out.
int enqueue_exhaustive(DevCtx* c, cudaStream_t st, const double* d_durs, int n, int dma,
                       double sigma, uint64_t lo, uint64_t hi, int fast, osim_summary* d_out,
                       double* d_ms, Part* parts, int max_parts, double thr = -HUGE_VAL,
                       unsigned long long* d_below = nullptr) {
    int g = 1;
    int rc = 0;
    if (hi > lo) {
        if (fast == 1) {  // the kernel's last CTA writes d_out (no final-reduce launch)
            rc = launch_exh_fast_dispatch(dma, n, c, st, d_durs, sigma, lo, hi, thr, parts, max_parts, d_ms, &g,
                                          d_out, d_below);
            if (rc) return rc;
            CK(cudaGetLastError());
            return 0;
        } else if (fast == 2) {  // null stages in the fast range: NullSim with prefix sharing
            if (null_pfx_launch(n, dma, sigma_pow2(sigma), LaunchCfg{c->sms, st}, d_durs, sigma, lo, hi, thr, parts,
                                max_parts, d_ms, c->d_err, &g))
                return fail(OSIM_EINVAL, "unsupported n=%d", n);
        } else {
            uint64_t blocks = (hi - lo + kBlock - 1) / kBlock;
            if (dma == 2) {
                g = grid_for(k_exhaustive_gen<2>, kBlock, 0, c, blocks);
                if (g > max_parts) g = max_parts;
                k_exhaustive_gen<2><<<g, kBlock, 0, st>>>(d_durs, n, sigma, lo, hi, thr, parts, d_ms, c->d_err);
            } else {
                g = grid_for(k_exhaustive_gen<1>, kBlock, 0, c, blocks);
                if (g > max_parts) g = max_parts;
                k_exhaustive_gen<1><<<g, kBlock, 0, st>>>(d_durs, n, sigma, lo, hi, thr, parts, d_ms, c->d_err);
            }
        }
        if (rc) return rc;
    } else {
        g = 0;
    }
    k_final_reduce<<<1, kBlock, 0, st>>>(parts, g, d_out, d_below);
    CK(cudaGetLastError());
    return 0;
}

int max_parts_for(const DevCtx* c) { return c->sms * 16; }

int enqueue_batch(DevCtx* c, cudaStream_t st, const double* d_durs, uint64_t B, int n, int dma,
                  double sigma, int fast, osim_summary* d_out) {
    if (B == 0) return 0;
    int rc = 0;
    if (fast == 1) {
        rc = launch_batch_fast_dispatch(dma, n, c, st, d_durs, B, sigma, d_out);
    } else if (fast == 2) {
        int g = 0;
        if (null_batch_launch(n, dma, sigma_pow2(sigma), LaunchCfg{c->sms, st}, d_durs, B, sigma, d_out, c->d_err, &g))
            return fail(OSIM_EINVAL, "unsupported n=%d", n);
    } else if (dma == 2) {
        int g = grid_for(k_exhaustive_batch_gen<2>, kBlock, 0, c, B);
        k_exhaustive_batch_gen<2><<<g, kBlock, 0, st>>>(d_durs, B, n, sigma, d_out, c->d_err);
    } else {
        int g = grid_for(k_exhaustive_batch_gen<1>, kBlock, 0, c, B);
        k_exhaustive_batch_gen<1><<<g, kBlock, 0, st>>>(d_durs, B, n, sigma, d_out, c->d_err);
    }
    if (rc) return rc;
    CK(cudaGetLastError());
    return 0;
}

int enqueue_heuristic(DevCtx* c, cudaStream_t st, const double* d_durs, const uint8_t* d_idr,
                      uint64_t B, int n, int dma, double sigma, int sum_mode, int fast,
                      uint8_t* d_order, double* d_ms, uint32_t* d_ns) {
    if (B == 0) return 0;
    if ((B + kHG - 1) / kHG > 0x7fffffffull) return fail(OSIM_EINVAL, "batch too large");
    // the launcher's temporaries (the lane kernel's group order): one buffer
    // per library stream, so the host path's two chunk streams never share one
    AuxBuf* aux = &c->aux[st == c->stream2 ? 1 : 0];
    heuristic_launch(dma, fast, LaunchCfg{c->sms, st, aux}, d_durs, d_idr, B, n, sigma, sum_mode, d_order, d_ms,
                     d_ns, c->d_err);
    CK(cudaGetLastError());
    return 0;
}

// Sync the device's stream and surface a kernel-side stall flag.
int finish(DevCtx* c, cudaStream_t st) {
    CK(cudaStreamSynchronize(st));
    int h_err = 0;
    CK(cudaMemcpy(&h_err, c->d_err, sizeof(int), cudaMemcpyDeviceToHost));
    if (h_err) {
        CK(cudaMemset(c->d_err, 0, sizeof(int)));
        return fail(h_err, "simulation stalled with commands pending");
    }
    return 0;
}

// Null stages allowed: every stage 0 or in the FastSim range (NullSim path).
bool null_fast_ok(const double* durs, uint64_t tasks, double sigma) {
    const double lo = std::ldexp(1.0, -60), hi = std::ldexp(1.0, 22);
    if (!(sigma >= lo)) return false;
    for (uint64_t i = 0; i < 3 * tasks; ++i)
        if (!(durs[i] == 0.0 || (durs[i] >= lo && durs[i] < hi))) return false;
    return true;
}

bool fast_ok(const double* durs, uint64_t tasks, double sigma) {
    const double lo = std::ldexp(1.0, -60), hi = std::ldexp(1.0, 22);  // kFastHi
    if (!(sigma >= lo)) return false;
    for (uint64_t i = 0; i < 3 * tasks; ++i)
        if (!(durs[i] >= lo && durs[i] < hi)) return false;
    return true;
}

void merge_host(osim_summary& a, const osim_summary& b) {
    if (b.count == 0) return;
    if (a.count == 0) { a = b; return; }
    if (b.best < a.best || (b.best == a.best && b.best_rank < a.best_rank)) {
        a.best = b.best;
        a.best_rank = b.best_rank;
    }
    if (b.worst > a.worst) a.worst = b.worst;
    a.sum += b.sum;
    a.sum_log += b.sum_log;
    a.count += b.count;
}

struct DevList {
    std::vector<DevCtx*> v;
};

int pick_devs(int n_dev, DevList& out) {
    int rc = ensure_init();
    if (rc) return rc;
    if (n_dev <= 1) {
        int d = cur_dev();
        if (d < 0 || d >= (int)g_devs.size()) return fail(OSIM_ENODEV, "device %d not available", d);
        out.v.push_back(g_devs[d]);
        return 0;
    }
    if (n_dev > (int)g_devs.size())
        return fail(OSIM_ENODEV, "requested %d devices, %d available", n_dev, (int)g_devs.size());
    for (int d = 0; d < n_dev; ++d) out.v.push_back(g_devs[d]);
    return 0;
}


// k-th smallest (0-based) of the positive doubles held by several devices
// (each device: d_vals[i] with counts[i] values); histograms of every pass
// are summed over devices on the host.  Exact: the result is a bit pattern.
// k-th smallest (0-based) of the values spread over the devices, by MSB-first
// radix selection on the bit patterns (positive doubles order like their
// bits).  The walk starts below the bits shared by the smallest and largest
// value (vmin, vmax: the summary's best / worst), and once the candidates
// fit the per-device compaction buffers (cbuf, ccap values each) the next
// pass also copies them out, so the remaining passes read only those.
// *same_next: whether the (k+1)-th value equals the k-th.
// Grid of k_radix_hist over `count` values: 8 CTAs per SM, more if a CTA
// would otherwise visit 2^32 values or more (its shared counts are 32-bit).
int radix_grid(uint64_t count, int sms) {
    const uint64_t blocks = (count + 255) / 256;
    uint64_t g = blocks < (uint64_t)sms * 8 ? blocks : (uint64_t)sms * 8;
    const uint64_t per_cta_max = (1ull << 32) - 256;  // values one CTA may visit
    while (g < blocks && ((count + g * 256 - 1) / (g * 256)) * 256 > per_cta_max) g *= 2;
    if (g > blocks) g = blocks;
    return (int)(g < 1 ? 1 : g);
}

int select_kth(std::vector<DevCtx*>& devs, std::vector<const double*>& vals, std::vector<uint64_t>& counts,
               std::vector<unsigned long long*>& d_hist, uint64_t k, double vmin, double vmax,
               std::vector<unsigned long long*>& cbuf, uint64_t ccap, double* out, bool* same_next) {
    unsigned long long prefix = 0, a, b;
    memcpy(&a, &vmin, sizeof(a));
    memcpy(&b, &vmax, sizeof(b));
    int pbits = 0;
    if (vmin > 0.0 && vmax >= vmin)  // common leading bits of every value in [vmin, vmax]
        while (pbits < 63 && ((a ^ b) >> (63 - pbits)) == 0) ++pbits;
    prefix = pbits ? (a >> (64 - pbits)) : 0ull;
    std::vector<const unsigned long long*> cur(devs.size());
    std::vector<uint64_t> cnt(counts);
    for (size_t i = 0; i < devs.size(); ++i) cur[i] = (const unsigned long long*)vals[i];
    uint64_t matching = 0;  // values carrying the current prefix, over all devices
    for (size_t i = 0; i < devs.size(); ++i) matching += cnt[i];
    bool compacted = false;
    std::vector<unsigned long long> h(1 << kRadixBits), tot(1 << kRadixBits);  // 64-bit: bins can exceed 2^32
    uint64_t last_bin_count = 0;
    while (pbits < 64) {
        const int d = (64 - pbits) < kRadixBits ? (64 - pbits) : kRadixBits;
        const int nb = 1 << d;
        const bool append = !compacted && pbits > 0 && matching <= ccap && !cbuf.empty();
        std::fill(tot.begin(), tot.begin() + nb, 0ull);
        std::vector<unsigned long long> got(devs.size(), 0);
        for (size_t i = 0; i < devs.size(); ++i) {
            DevCtx* c = devs[i];
            CK(cudaSetDevice(c->dev));
            CK(cudaMemsetAsync(d_hist[i], 0, nb * sizeof(unsigned long long), c->stream));
            unsigned long long* d_cnt = d_hist[i] + (1u << kRadixBits);
            if (append) CK(cudaMemsetAsync(d_cnt, 0, sizeof(unsigned long long), c->stream));
            if (cnt[i]) {
                const int g = radix_grid(cnt[i], c->sms);
                k_radix_hist<<<g, 256, 0, c->stream>>>(cur[i], cnt[i], prefix, pbits, d, d_hist[i],
                                                       append ? cbuf[i] : nullptr, append ? d_cnt : nullptr);
                CK(cudaGetLastError());
            }
            CK(cudaMemcpyAsync(h.data(), d_hist[i], nb * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                               c->stream));
            if (append) CK(cudaMemcpyAsync(&got[i], d_cnt, sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream));
            CK(cudaStreamSynchronize(c->stream));
            for (int bb = 0; bb < nb; ++bb) tot[bb] += h[bb];
        }
        if (append) {
            for (size_t i = 0; i < devs.size(); ++i) { cur[i] = cbuf[i]; cnt[i] = got[i]; }
            compacted = true;
        }
        uint64_t cum = 0;
        int bin = 0;
        for (; bin < nb; ++bin) {
            if (cum + tot[bin] > k) break;
            cum += tot[bin];
        }
        if (bin == nb) return fail(OSIM_EINVAL, "rank %llu outside the value set", (unsigned long long)k);
        k -= cum;
        matching = tot[bin];
        last_bin_count = tot[bin];
        prefix = (prefix << d) | (unsigned long long)bin;
        pbits += d;
    }
    double v;
    memcpy(&v, &prefix, sizeof(v));
    *out = v;
    if (same_next) *same_next = k + 1 < last_bin_count;  // v occurs again at rank k + 1
    return 0;
}
}  // namespace

// Groups of 17..64 tasks (osim_wide.cuh): validated on the host, one
// group per thread on the general path, sharded over devices by group range.
int heuristic_wide(const double* durs, const uint8_t* id_rank, uint64_t B, int n, int dma, double sigma,
                   int sum_mode, int n_dev, uint8_t* order, double* makespan, uint32_t* n_sims) {
    int rc = check_common(n, dma, sigma, kWideMaxN);
    if (rc) return rc;
    if (B && (!durs || !id_rank || !order || !makespan)) return fail(OSIM_EINVAL, "NULL buffer");
    if ((rc = check_durs(durs, B * (uint64_t)n))) return rc;
    if ((rc = check_id_ranks(id_rank, B, n))) return rc;
    DevList dl;
    if ((rc = pick_devs(n_dev, dl))) return rc;
    const int G = (int)dl.v.size();
    std::vector<std::unique_lock<std::mutex>> locks;
    for (int gi = 0; gi < G; ++gi) {
        DevCtx* c = dl.v[gi];
        locks.emplace_back(c->mu);
        CK(cudaSetDevice(c->dev));
        const uint64_t lo = B * (uint64_t)gi / (uint64_t)G, hi = B * (uint64_t)(gi + 1) / (uint64_t)G;
        const uint64_t m = hi - lo;
        if (!m) continue;
        const size_t off_idr = align_up(m * 3 * n * sizeof(double));
        const size_t off_ord = off_idr + align_up(m * n);
        const size_t off_ms = off_ord + align_up(m * n);
        const size_t off_ns = off_ms + align_up(m * sizeof(double));
        void* base;
        if ((rc = scratch(c, off_ns + align_up(m * sizeof(uint32_t)), &base))) return rc;
        char* b = (char*)base;
        CK(cudaMemcpyAsync(b, durs + lo * 3 * n, m * 3 * n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(b + off_idr, id_rank + lo * n, m * n, cudaMemcpyHostToDevice, c->stream));
        wide_heuristic_launch(dma, LaunchCfg{c->sms, c->stream}, (double*)b, (uint8_t*)(b + off_idr), m, n, sigma,
                              sum_mode, (uint8_t*)(b + off_ord), (double*)(b + off_ms), (uint32_t*)(b + off_ns),
                              c->d_err);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(order + lo * n, b + off_ord, m * n, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(makespan + lo, b + off_ms, m * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        if (n_sims) CK(cudaMemcpyAsync(n_sims + lo, b + off_ns, m * sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
    }
    for (int gi = 0; gi < G; ++gi) {
        DevCtx* c = dl.v[gi];
        CK(cudaSetDevice(c->dev));
        if ((rc = finish(c, c->stream))) return rc;
    }
    return 0;
}

extern "C" {

const char* osim_version(void) { return "offsim-b200 0.1.0 (sm_100a)"; }
const char* osim_last_error(void) { return g_err.c_str(); }

int osim_init(int want_devices, int* got) {
    int rc = ensure_init();
    if (rc) return rc;
    int n = (int)g_devs.size();
    if (want_devices > 0 && want_devices < n) n = want_devices;
    if (got) *got = n;
    return 0;
}

int osim_shutdown(void) {
    std::lock_guard<std::mutex> lk(g_init_mu);
    for (DevCtx* c : g_devs) {
        cudaSetDevice(c->dev);
        cudaDeviceSynchronize();
        if (c->scratch) cudaFree(c->scratch);
        for (AuxBuf& a : c->aux) {
            if (a.p) cudaFree(a.p);
            if (a.ev) cudaEventDestroy(a.ev);
        }
        if (c->d_err) cudaFree(c->d_err);
        if (c->d_done) cudaFree(c->d_done);
        if (c->stream) cudaStreamDestroy(c->stream);
        if (c->stream2) cudaStreamDestroy(c->stream2);
        if (c->ev) cudaEventDestroy(c->ev);
        delete c;
    }
    g_devs.clear();
    return 0;
}

int osim_set_device(int device) {
    int rc = ensure_init();
    if (rc) return rc;
    if (device < 0 || device >= (int)g_devs.size())
        return fail(OSIM_ENODEV, "device %d not available (%d visible)", device, (int)g_devs.size());
    g_thread_dev = device;
    CK(cudaSetDevice(g_devs[device]->dev));
    return 0;
}

int osim_fast_eligible(const double* durs, uint64_t count, double sigma) {
    if (!durs) return 0;
    return fast_ok(durs, count, sigma) ? 1 : 0;
}

int osim_pfx_suffix_len(int n) {
    if (n < 1 || n > kMaxN) return fail(OSIM_EINVAL, "n=%d outside [1, %d]", n, kMaxN);
    return pfx_l_for(n);
}

int osim_exhaustive(const double* durs, int n, int dma, double sigma, uint64_t rank_lo,
                    uint64_t rank_hi, int n_dev, osim_summary* out, double* makespans) {
    int rc = check_common(n, dma, sigma);
    if (rc) return rc;
    if (n > 20) return fail(OSIM_EINVAL, "n too large for 64-bit ranks");
    if ((rc = check_durs(durs, (uint64_t)n))) return rc;
    if (!out) return fail(OSIM_EINVAL, "out is NULL");
    const uint64_t total = factorial(n);
    if (rank_lo > rank_hi || rank_hi > total)
        return fail(OSIM_EINVAL, "rank range [%llu, %llu) outside [0, %llu)", (unsigned long long)rank_lo,
                    (unsigned long long)rank_hi, (unsigned long long)total);
    DevList dl;
    if ((rc = pick_devs(n_dev, dl))) return rc;
    const int fast = fast_ok(durs, n, sigma) ? 1 : (null_fast_ok(durs, n, sigma) ? 2 : 0);
    const int G = (int)dl.v.size();
    const uint64_t span = rank_hi - rank_lo;
    std::vector<osim_summary> res(G);
    std::vector<std::unique_lock<std::mutex>> locks;
    // enqueue on every device, then collect in device order
    for (int gi = 0; gi < G; ++gi) {
        DevCtx* c = dl.v[gi];
        locks.emplace_back(c->mu);
        CK(cudaSetDevice(c->dev));
        const uint64_t lo = rank_lo + span * (uint64_t)gi / (uint64_t)G;
        const uint64_t hi = rank_lo + span * (uint64_t)(gi + 1) / (uint64_t)G;
        const int mp = max_parts_for(c);
        size_t off_parts = align_up(3 * kMaxN * sizeof(double));
        size_t off_sum = off_parts + align_up(mp * sizeof(Part));
        size_t off_ms = off_sum + align_up(sizeof(osim_summary));
        size_t bytes = off_ms + (makespans ? align_up((hi - lo) * sizeof(double)) : 0);
        void* base;
        if ((rc = scratch(c, bytes, &base))) return rc;
        char* b = (char*)base;
        CK(cudaMemcpyAsync(b, durs, 3 * n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        double* d_ms = makespans ? (double*)(b + off_ms) : nullptr;
        rc = enqueue_exhaustive(c, c->stream, (double*)b, n, dma, sigma, lo, hi, fast,
                                (osim_summary*)(b + off_sum), d_ms, (Part*)(b + off_parts), mp);
        if (rc) return rc;
        CK(cudaMemcpyAsync(&res[gi], b + off_sum, sizeof(osim_summary), cudaMemcpyDeviceToHost, c->stream));
        if (makespans)
            CK(cudaMemcpyAsync(makespans + (lo - rank_lo), d_ms, (hi - lo) * sizeof(double),
                               cudaMemcpyDeviceToHost, c->stream));
    }
    osim_summary acc;
    memset(&acc, 0, sizeof(acc));
    for (int gi = 0; gi < G; ++gi) {
        DevCtx* c = dl.v[gi];
        CK(cudaSetDevice(c->dev));
        if ((rc = finish(c, c->stream))) return rc;
        merge_host(acc, res[gi]);
    }
    *out = acc;
    return 0;
}

int osim_exhaustive_dev(const double* d_durs, int n, int dma, double sigma, uint64_t rank_lo,
                        uint64_t rank_hi, int fast, osim_summary* d_out, double* d_makespans,
                        void* stream) {
    int rc = check_common(n, dma, sigma);
    if (rc) return rc;
    if (rank_lo > rank_hi || rank_hi > factorial(n)) return fail(OSIM_EINVAL, "bad rank range");
    DevList dl;
    if ((rc = pick_devs(1, dl))) return rc;
    DevCtx* c = dl.v[0];
    std::lock_guard<std::mutex> lk(c->mu);
    cudaStream_t st = stream ? (cudaStream_t)stream : c->stream;
    const int mp = max_parts_for(c);
    void* base;
    if ((rc = scratch(c, align_up(mp * sizeof(Part)), &base))) return rc;
    return enqueue_exhaustive(c, st, d_durs, n, dma, sigma, rank_lo, rank_hi, fast, d_out,
                              d_makespans, (Part*)base, mp);
}

// one shard of [0, n!) (see offsim_b200.h): interleaved 512-prefix calls on
// the fast path, the contiguous range otherwise
int enqueue_shard(DevCtx* c, cudaStream_t st, const double* d_durs, int n, int dma, double sigma, int shard,
                  int shards, int fast, osim_summary* d_out, Part* parts, int mp) {
    const uint64_t total = factorial(n);
    if (fast == 1) {
        int g = 1;
        int rc = launch_exh_fast_dispatch(dma, n, c, st, d_durs, sigma, 0, total, -HUGE_VAL, parts, mp, nullptr, &g,
                                          d_out, nullptr, (unsigned)shard, (unsigned)shards);
        if (rc) return rc;
        CK(cudaGetLastError());
        return 0;
    }
    const uint64_t lo = (uint64_t)((unsigned __int128)total * (unsigned)shard / (unsigned)shards);
    const uint64_t hi = (uint64_t)((unsigned __int128)total * (unsigned)(shard + 1) / (unsigned)shards);
    return enqueue_exhaustive(c, st, d_durs, n, dma, sigma, lo, hi, fast, d_out, nullptr, parts, mp);
}

int osim_exhaustive_shard_dev(const double* d_durs, int n, int dma, double sigma, int shard, int shards, int fast,
                              osim_summary* d_out, void* stream) {
    int rc = check_common(n, dma, sigma);
    if (rc) return rc;
    if (shards < 1 || shard < 0 || shard >= shards) return fail(OSIM_EINVAL, "shard %d of %d", shard, shards);
    DevList dl;
    if ((rc = pick_devs(1, dl))) return rc;
    DevCtx* c = dl.v[0];
    std::lock_guard<std::mutex> lk(c->mu);
    cudaStream_t st = stream ? (cudaStream_t)stream : c->stream;
    const int mp = max_parts_for(c);
    void* base;
    if ((rc = scratch(c, align_up(mp * sizeof(Part)), &base))) return rc;
    return enqueue_shard(c, st, d_durs, n, dma, sigma, shard, shards, fast, d_out, (Part*)base, mp);
}

int osim_exhaustive_shard(const double* durs, int n, int dma, double sigma, int shard, int shards,
                          osim_summary* out) {
    int rc = check_common(n, dma, sigma);
    if (rc) return rc;
    if ((rc = check_durs(durs, (uint64_t)n))) return rc;
    if (!out) return fail(OSIM_EINVAL, "out is NULL");
    if (shards < 1 || shard < 0 || shard >= shards) return fail(OSIM_EINVAL, "shard %d of %d", shard, shards);
    DevList dl;
    if ((rc = pick_devs(1, dl))) return rc;
    DevCtx* c = dl.v[0];
    std::lock_guard<std::mutex> lk(c->mu);
    const int fast = fast_ok(durs, n, sigma) ? 1 : (null_fast_ok(durs, n, sigma) ? 2 : 0);
    const int mp = max_parts_for(c);
    const size_t off_parts = align_up(3 * kMaxN * sizeof(double));
    const size_t off_sum = off_parts + align_up(mp * sizeof(Part));
    void* base;
    if ((rc = scratch(c, off_sum + align_up(sizeof(osim_summary)), &base))) return rc;
    char* b = (char*)base;
    CK(cudaMemcpyAsync(b, durs, 3 * n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    if ((rc = enqueue_shard(c, c->stream, (double*)b, n, dma, sigma, shard, shards, fast, (osim_summary*)(b + off_sum),
                            (Part*)(b + off_parts), mp)))
        return rc;
    CK(cudaMemcpyAsync(out, b + off_sum, sizeof(osim_summary), cudaMemcpyDeviceToHost, c->stream));
    return finish(c, c->stream);
}

int osim_exhaustive_stats(const double* durs, int n, int dma, double sigma, uint64_t rank_lo, uint64_t rank_hi,
                          double threshold, int n_dev, osim_summary* out, uint64_t* below, double* median) {
    int rc = check_common(n, dma, sigma);
    if (rc) return rc;
    if ((rc = check_durs(durs, (uint64_t)n))) return rc;
    if (!out) return fail(OSIM_EINVAL, "out is NULL");
    const uint64_t total = factorial(n);
    if (rank_lo > rank_hi || rank_hi > total) return fail(OSIM_EINVAL, "bad rank range");
    DevList dl;
    if ((rc = pick_devs(n_dev, dl))) return rc;
    const int fast = fast_ok(durs, n, sigma) ? 1 : (null_fast_ok(durs, n, sigma) ? 2 : 0);
    const int G = (int)dl.v.size();
    const uint64_t span = rank_hi - rank_lo;
    std::vector<osim_summary> res(G);
    std::vector<unsigned long long> bel(G, 0);
    std::vector<const double*> vals(G);
    std::vector<uint64_t> counts(G);
    std::vector<unsigned long long*> hists(G);
    std::vector<unsigned long long*> cbufs(G);
    uint64_t ccap = 0;  // per-device compaction capacity (values)
    std::vector<std::unique_lock<std::mutex>> locks;
    for (int gi = 0; gi < G; ++gi) {
        DevCtx* c = dl.v[gi];
        locks.emplace_back(c->mu);
        CK(cudaSetDevice(c->dev));
        const uint64_t lo = rank_lo + span * (uint64_t)gi / (uint64_t)G;
        const uint64_t hi = rank_lo + span * (uint64_t)(gi + 1) / (uint64_t)G;
        const int mp = max_parts_for(c);
        size_t off_parts = align_up(3 * kMaxN * sizeof(double));
        size_t off_sum = off_parts + align_up(mp * sizeof(Part));
        size_t off_bel = off_sum + align_up(sizeof(osim_summary));
        size_t off_hist = off_bel + 256;
        size_t off_ms = off_hist + align_up(((1u << kRadixBits) + 1) * sizeof(unsigned long long));
        size_t off_cb = off_ms + align_up((hi - lo) * sizeof(double) + 8);
        size_t bytes = off_cb + (median ? align_up(((hi - lo) / 8 + 1) * sizeof(double)) : 0);
        void* base;
        if ((rc = scratch(c, bytes, &base))) return rc;
        char* b = (char*)base;
        CK(cudaMemcpyAsync(b, durs, 3 * n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        rc = enqueue_exhaustive(c, c->stream, (double*)b, n, dma, sigma, lo, hi, fast, (osim_summary*)(b + off_sum),
                                (double*)(b + off_ms), (Part*)(b + off_parts), mp, threshold,
                                (unsigned long long*)(b + off_bel));
        if (rc) return rc;
        CK(cudaMemcpyAsync(&res[gi], b + off_sum, sizeof(osim_summary), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(&bel[gi], b + off_bel, sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream));
        vals[gi] = (const double*)(b + off_ms);
        counts[gi] = hi - lo;
        hists[gi] = (unsigned long long*)(b + off_hist);
        cbufs[gi] = (unsigned long long*)(b + off_cb);
        ccap = (gi == 0 || (hi - lo) / 8 + 1 < ccap) ? (hi - lo) / 8 + 1 : ccap;
    }
    osim_summary acc;
    memset(&acc, 0, sizeof(acc));
    uint64_t nbelow = 0;
    for (int gi = 0; gi < G; ++gi) {
        DevCtx* c = dl.v[gi];
        CK(cudaSetDevice(c->dev));
        if ((rc = finish(c, c->stream))) return rc;
        merge_host(acc, res[gi]);
        nbelow += bel[gi];
    }
    *out = acc;
    if (below) *below = nbelow;
    if (median) {
        // np.median (numpy/lib/function_base.py): the middle value, or for an
        // even count the mean of the two middle values, (a + b) / 2
        const uint64_t cnt = acc.count;
        if (cnt == 0) {
            *median = NAN;
        } else if (cnt & 1) {
            if ((rc = select_kth(dl.v, vals, counts, hists, cnt / 2, acc.best, acc.worst, cbufs, ccap, median,
                                 nullptr)))
                return rc;
        } else {
            double a, bb;
            bool same = false;
            if ((rc = select_kth(dl.v, vals, counts, hists, cnt / 2 - 1, acc.best, acc.worst, cbufs, ccap, &a,
                                 &same)))
                return rc;
            if (same) bb = a;  // the two middle values are equal
            else if ((rc = select_kth(dl.v, vals, counts, hists, cnt / 2, acc.best, acc.worst, cbufs, ccap, &bb,
                                      nullptr)))
                return rc;
            volatile double s = a + bb;  // two IEEE roundings, as numpy's mean
            *median = s / 2.0;
        }
    }
    for (DevCtx* c : dl.v) trim_scratch(c);
    return 0;
}

int osim_radix_hist_dev(const double* d_vals, uint64_t count, uint64_t prefix, int prefix_bits, int digit_bits,
                        uint64_t* d_hist, void* stream) {
    if (prefix_bits < 0 || digit_bits < 1 || digit_bits > kRadixBits || prefix_bits + digit_bits > 64)
        return fail(OSIM_EINVAL, "bad radix digit (prefix %d bits, digit %d bits)", prefix_bits, digit_bits);
    DevList dl;
    int rc = pick_devs(1, dl);
    if (rc) return rc;
    DevCtx* c = dl.v[0];
    cudaStream_t st = stream ? (cudaStream_t)stream : c->stream;
    CK(cudaMemsetAsync(d_hist, 0, (1u << digit_bits) * sizeof(uint64_t), st));
    if (count) {
        const int g = radix_grid(count, c->sms);
        k_radix_hist<<<g, 256, 0, st>>>((const unsigned long long*)d_vals, count, prefix, prefix_bits, digit_bits,
                                        (unsigned long long*)d_hist);
    }
    CK(cudaGetLastError());
    return 0;
}

int osim_select_kth_dev(const double* d_vals, uint64_t count, uint64_t k, double* kth, void* stream) {
    if (!kth) return fail(OSIM_EINVAL, "kth is NULL");
    if (count && !d_vals) return fail(OSIM_EINVAL, "d_vals is NULL");
    if (k >= count) return fail(OSIM_EINVAL, "rank %llu outside [0, %llu)", (unsigned long long)k,
                                (unsigned long long)count);
    DevList dl;
    int rc = pick_devs(1, dl);
    if (rc) return rc;
    DevCtx* c = dl.v[0];
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->dev));
    if (stream) CK(cudaStreamSynchronize((cudaStream_t)stream));  // the values are complete
    void* base;
    if ((rc = scratch(c, align_up(((1u << kRadixBits) + 1) * sizeof(unsigned long long)), &base))) return rc;
    std::vector<const double*> vals{d_vals};
    std::vector<uint64_t> counts{count};
    std::vector<unsigned long long*> hists{(unsigned long long*)base};
    std::vector<unsigned long long*> nocb;
    return select_kth(dl.v, vals, counts, hists, k, 0.0, 0.0, nocb, 0, kth, nullptr);
}

int osim_exhaustive_ex_dev(const double* d_durs, int n, int dma, double sigma, uint64_t rank_lo, uint64_t rank_hi,
                           int fast, double threshold, osim_summary* d_out, uint64_t* d_below, double* d_makespans,
                           void* stream) {
    int rc = check_common(n, dma, sigma);
    if (rc) return rc;
    if (rank_lo > rank_hi || rank_hi > factorial(n)) return fail(OSIM_EINVAL, "bad rank range");
    DevList dl;
    if ((rc = pick_devs(1, dl))) return rc;
    DevCtx* c = dl.v[0];
    std::lock_guard<std::mutex> lk(c->mu);
    cudaStream_t st = stream ? (cudaStream_t)stream : c->stream;
    const int mp = max_parts_for(c);
    void* base;
    if ((rc = scratch(c, align_up(mp * sizeof(Part)), &base))) return rc;
    return enqueue_exhaustive(c, st, d_durs, n, dma, sigma, rank_lo, rank_hi, fast, d_out, d_makespans, (Part*)base,
                              mp, threshold, (unsigned long long*)d_below);
}

int osim_eval_perms(const double* durs, int n, int dma, double sigma, const uint8_t* perms,
                    uint64_t cnt, int n_dev, double* makespans, osim_summary* out) {
    int rc = check_common(n, dma, sigma, kWideMaxN);
    if (rc) return rc;
    if ((rc = check_durs(durs, (uint64_t)n))) return rc;
    if (!perms && cnt) return fail(OSIM_EINVAL, "perms is NULL");
    if (!makespans && cnt) return fail(OSIM_EINVAL, "makespans is NULL");
    for (uint64_t i = 0; i < cnt; ++i) {  // each row must be a permutation of range(n)
        uint64_t seen = 0;
        for (int j = 0; j < n; ++j) {
            const unsigned v = perms[i * n + j];
            if (v >= (unsigned)n || ((seen >> v) & 1ull))
                return fail(OSIM_EINVAL, "row %llu is not a permutation of range(%d)", (unsigned long long)i, n);
            seen |= 1ull << v;
        }
    }
    DevList dl;
    if ((rc = pick_devs(n_dev, dl))) return rc;
    const int fast = fast_ok(durs, n, sigma);
    const int G = (int)dl.v.size();
    std::vector<osim_summary> res(G);
    std::vector<std::unique_lock<std::mutex>> locks;
    for (int gi = 0; gi < G; ++gi) {
        DevCtx* c = dl.v[gi];
        locks.emplace_back(c->mu);
        CK(cudaSetDevice(c->dev));
        const uint64_t lo = cnt * (uint64_t)gi / (uint64_t)G, hi = cnt * (uint64_t)(gi + 1) / (uint64_t)G;
        const uint64_t m = hi - lo;
        const int mp = max_parts_for(c);
        size_t off_parts = align_up(3 * kWideMaxN * sizeof(double));
        size_t off_sum = off_parts + align_up(mp * sizeof(Part));
        size_t off_ms = off_sum + align_up(sizeof(osim_summary));
        size_t off_p = off_ms + align_up(m * sizeof(double) + 8);
        size_t bytes = off_p + align_up(m * n + 8);
        void* base;
        if ((rc = scratch(c, bytes, &base))) return rc;
        char* b = (char*)base;
        CK(cudaMemcpyAsync(b, durs, 3 * n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        if (m) CK(cudaMemcpyAsync(b + off_p, perms + lo * n, m * n, cudaMemcpyHostToDevice, c->stream));
        Part* parts = (Part*)(b + off_parts);
        int g = 0;
        if (m && n > kMaxN) {  // 17..64 tasks: the byte-FIFO general path
            const LaunchCfg cfg{c->sms, c->stream};
            g = wide_eval_perms_launch(dma, cfg, (double*)b, n, sigma, (uint8_t*)(b + off_p), m,
                                       (double*)(b + off_ms), parts, mp, c->d_err);
        } else if (m) {
            const uint64_t blocks = (m + kBlock - 1) / kBlock;
#define OSIM_EP(D, F)                                                                            \
    do {                                                                                         \
        g = grid_for(k_eval_perms<D, F>, kBlock, 0, c, blocks);                                  \
        if (g > mp) g = mp;                                                                      \
        k_eval_perms<D, F><<<g, kBlock, 0, c->stream>>>((double*)b, n, sigma, (uint8_t*)(b + off_p), m, -HUGE_VAL, \
                                                         (double*)(b + off_ms), parts, c->d_err); \
    } while (0)
            if (dma == 2) { if (fast) OSIM_EP(2, true); else OSIM_EP(2, false); }
            else { if (fast) OSIM_EP(1, true); else OSIM_EP(1, false); }
#undef OSIM_EP
        }
        k_final_reduce<<<1, kBlock, 0, c->stream>>>(parts, g, (osim_summary*)(b + off_sum), nullptr);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(&res[gi], b + off_sum, sizeof(osim_summary), cudaMemcpyDeviceToHost, c->stream));
        if (m) CK(cudaMemcpyAsync(makespans + lo, b + off_ms, m * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    }
    osim_summary acc;
    memset(&acc, 0, sizeof(acc));
    for (int gi = 0; gi < G; ++gi) {
        DevCtx* c = dl.v[gi];
        CK(cudaSetDevice(c->dev));
        if ((rc = finish(c, c->stream))) return rc;
        // device-local indices -> list indices
        const uint64_t lo = cnt * (uint64_t)gi / (uint64_t)G;
        res[gi].best_rank += lo;
        merge_host(acc, res[gi]);
    }
    if (out) *out = acc;
    return 0;
}

int osim_exhaustive_batch(const double* durs, uint64_t B, int n, int dma, double sigma, int n_dev,
                          osim_summary* out) {
    int rc = check_common(n, dma, sigma);
    if (rc) return rc;
    if (n > 12) return fail(OSIM_EINVAL, "batched exhaustive search supports n <= 12");
    int fast = 0;
    if ((rc = scan_durs(durs, B * (uint64_t)n, sigma, &fast))) return rc;
    if (!out && B) return fail(OSIM_EINVAL, "out is NULL");
    DevList dl;
    if ((rc = pick_devs(n_dev, dl))) return rc;
    const int G = (int)dl.v.size();
    std::vector<std::unique_lock<std::mutex>> locks;
    for (int gi = 0; gi < G; ++gi) {
        DevCtx* c = dl.v[gi];
        locks.emplace_back(c->mu);
        CK(cudaSetDevice(c->dev));
        const uint64_t lo = B * (uint64_t)gi / (uint64_t)G, hi = B * (uint64_t)(gi + 1) / (uint64_t)G;
        const uint64_t m = hi - lo;
        size_t off_out = align_up(m * 3 * n * sizeof(double) + 8);
        size_t bytes = off_out + align_up(m * sizeof(osim_summary) + 8);
        void* base;
        if ((rc = scratch(c, bytes, &base))) return rc;
        char* b = (char*)base;
        if (m) {
            CK(cudaMemcpyAsync(b, durs + lo * 3 * n, m * 3 * n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
            if ((rc = enqueue_batch(c, c->stream, (double*)b, m, n, dma, sigma, fast, (osim_summary*)(b + off_out))))
                return rc;
            CK(cudaMemcpyAsync(out + lo, b + off_out, m * sizeof(osim_summary), cudaMemcpyDeviceToHost, c->stream));
        }
    }
    for (int gi = 0; gi < G; ++gi) {
        DevCtx* c = dl.v[gi];
        CK(cudaSetDevice(c->dev));
        if ((rc = finish(c, c->stream))) return rc;
    }
    return 0;
}

int osim_exhaustive_batch_dev(const double* d_durs, uint64_t B, int n, int dma, double sigma,
                              int fast, osim_summary* d_out, void* stream) {
    int rc = check_common(n, dma, sigma);
    if (rc) return rc;
    if (n > 12) return fail(OSIM_EINVAL, "batched exhaustive search supports n <= 12");
    DevList dl;
    if ((rc = pick_devs(1, dl))) return rc;
    DevCtx* c = dl.v[0];
    std::lock_guard<std::mutex> lk(c->mu);
    return enqueue_batch(c, stream ? (cudaStream_t)stream : c->stream, d_durs, B, n, dma, sigma, fast, d_out);
}

int osim_heuristic_batch(const double* durs, const uint8_t* id_rank, uint64_t B, int n, int dma,
                         double sigma, int sum_mode, int n_dev, uint8_t* order, double* makespan,
                         uint32_t* n_sims) {
    if (n > kMaxN) return heuristic_wide(durs, id_rank, B, n, dma, sigma, sum_mode, n_dev, order, makespan, n_sims);
    int rc = check_common(n, dma, sigma);
    if (rc) return rc;
    if (B && (!durs || !id_rank || !order || !makespan)) return fail(OSIM_EINVAL, "NULL buffer");
    DevList dl;
    if ((rc = pick_devs(n_dev, dl))) return rc;
    const int G = (int)dl.v.size();
    std::vector<std::unique_lock<std::mutex>> locks;
    std::vector<unsigned long long*> d_chk(G, nullptr);
    std::vector<char*> bases(G, nullptr);
    std::vector<uint64_t> los(G), ms_(G);
    std::vector<size_t> offs_idr(G), offs_ord(G), offs_ms(G), offs_ns(G);
    const bool fast_first = sigma >= 0x1p-60;
    // Inputs are validated on the device (a check kernel per chunk) while the
    // fast kernel runs optimistically on them -- it is memory-safe for any
    // values; a batch that turns out not to be fast-eligible is re-run through
    // the general kernel, and invalid input returns the reference's error.
    for (int gi = 0; gi < G; ++gi) {
        DevCtx* c = dl.v[gi];
        locks.emplace_back(c->mu);
        CK(cudaSetDevice(c->dev));
        const uint64_t lo = B * (uint64_t)gi / (uint64_t)G, hi = B * (uint64_t)(gi + 1) / (uint64_t)G;
        const uint64_t m = hi - lo;
        los[gi] = lo;
        ms_[gi] = m;
        if (!m) continue;
        size_t off_chk = align_up(m * 3 * n * sizeof(double));
        size_t off_idr = off_chk + 256;
        size_t off_ord = off_idr + align_up(m * n);
        size_t off_ms = off_ord + align_up(m * n);
        size_t off_ns = off_ms + align_up(m * sizeof(double));
        size_t bytes = off_ns + align_up(m * sizeof(uint32_t));
        void* base;
        if ((rc = scratch(c, bytes, &base))) return rc;
        char* b = (char*)base;
        bases[gi] = b;
        offs_idr[gi] = off_idr; offs_ord[gi] = off_ord; offs_ms[gi] = off_ms; offs_ns[gi] = off_ns;
        unsigned long long* chk = (unsigned long long*)(b + off_chk);
        d_chk[gi] = chk;
        const unsigned long long init[4] = {~0ull, ~0ull, 0ull, 0ull};
        CK(cudaMemcpyAsync(chk, init, sizeof(init), cudaMemcpyHostToDevice, c->stream));
        CK(cudaStreamSynchronize(c->stream));  // `init` is a stack buffer
        CK(cudaEventRecord(c->ev, c->stream));
        CK(cudaStreamWaitEvent(c->stream2, c->ev, 0));
        // large batches: chunks alternate between two streams so the H2D of
        // chunk i+1 and the D2H of chunk i-1 overlap the kernel of chunk i
        // (effective when the caller's buffers are pinned)
        static const uint64_t kChunks = [] {  // OSIM_HCHUNKS overrides (tuning only)
            const char* e = std::getenv("OSIM_HCHUNKS");
            const int x = e ? std::atoi(e) : 0;
            return (uint64_t)((x >= 1 && x <= 256) ? x : 8);
        }();
        const uint64_t nchunk = m >= (1ull << 17) ? kChunks : 1;
        for (uint64_t ci = 0; ci < nchunk; ++ci) {
            const uint64_t a = m * ci / nchunk, e = m * (ci + 1) / nchunk, mm = e - a;
            if (!mm) continue;
            cudaStream_t st = (ci & 1) ? c->stream2 : c->stream;
            double* d_durs = (double*)b + a * 3 * n;
            uint8_t* d_idr = (uint8_t*)(b + off_idr) + a * n;
            uint8_t* d_ord = (uint8_t*)(b + off_ord) + a * n;
            double* d_ms = (double*)(b + off_ms) + a;
            uint32_t* d_ns = (uint32_t*)(b + off_ns) + a;
            CK(cudaMemcpyAsync(d_durs, durs + (lo + a) * 3 * n, mm * 3 * n * sizeof(double),
                               cudaMemcpyHostToDevice, st));
            CK(cudaMemcpyAsync(d_idr, id_rank + (lo + a) * n, mm * n, cudaMemcpyHostToDevice, st));
            const unsigned cg = (unsigned)((mm + 255) / 256 < (uint64_t)c->sms * 4 ? (mm + 255) / 256 : c->sms * 4);
            k_check_batch<<<cg, 256, 0, st>>>(d_durs, d_idr, mm, n, (lo + a) * n, lo + a, chk);
            if ((rc = enqueue_heuristic(c, st, d_durs, d_idr, mm, n, dma, sigma, sum_mode, fast_first, d_ord, d_ms, d_ns)))
                return rc;
            CK(cudaMemcpyAsync(order + (lo + a) * n, d_ord, mm * n, cudaMemcpyDeviceToHost, st));
            CK(cudaMemcpyAsync(makespan + lo + a, d_ms, mm * sizeof(double), cudaMemcpyDeviceToHost, st));
            if (n_sims)
                CK(cudaMemcpyAsync(n_sims + lo + a, d_ns, mm * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
        }
    }
    // every device's streams are drained (and its error flag reset after an
    // optimistic pass over ineligible data) before any error is returned, so
    // no copy into the caller's buffers is still in flight
    std::vector<std::array<unsigned long long, 4>> chk(G);
    int sync_rc = 0;
    for (int gi = 0; gi < G; ++gi) {
        DevCtx* c = dl.v[gi];
        chk[gi] = {~0ull, ~0ull, 0ull, 0ull};
        if (!ms_[gi]) continue;
        if (cudaSetDevice(c->dev) != cudaSuccess || cudaStreamSynchronize(c->stream2) != cudaSuccess ||
            cudaStreamSynchronize(c->stream) != cudaSuccess ||
            cudaMemcpy(chk[gi].data(), d_chk[gi], sizeof(chk[gi]), cudaMemcpyDeviceToHost) != cudaSuccess) {
            if (!sync_rc) sync_rc = fail(OSIM_ECUDA, "device %d: %s", c->dev, cudaGetErrorString(cudaGetLastError()));
            continue;
        }
        const auto& res = chk[gi];
        if (res[0] != ~0ull || res[1] != ~0ull || (fast_first && res[2]))
            cudaMemset(c->d_err, 0, sizeof(int));  // the optimistic pass ran on ineligible data
    }
    if (sync_rc) return sync_rc;
    for (int gi = 0; gi < G; ++gi) {
        const auto& res = chk[gi];
        if (res[0] != ~0ull) {  // the reason, for the reference's message
            const uint64_t t = res[0];
            const double* d = durs + 3 * t;
            if (d[0] == 0.0 && d[1] == 0.0 && d[2] == 0.0)
                return fail(OSIM_EINVAL, "task %llu has no commands", (unsigned long long)t);
            return fail(OSIM_EINVAL, "task %llu: durations must be finite and non-negative", (unsigned long long)t);
        }
        if (res[1] != ~0ull)
            return fail(OSIM_EINVAL, "group %llu: id ranks must be a permutation (duplicate task id?)", res[1]);
    }
    for (int gi = 0; gi < G; ++gi) {
        DevCtx* c = dl.v[gi];
        const auto& res = chk[gi];
        if (!ms_[gi] || !(fast_first && res[2])) continue;
        CK(cudaSetDevice(c->dev));
        // not fast-eligible: recompute this shard with the null-stage kernel
        // (every stage 0 or in range) or the general one
        const uint64_t m = ms_[gi];
        char* b = bases[gi];
        if ((rc = enqueue_heuristic(c, c->stream, (double*)b, (uint8_t*)(b + offs_idr[gi]), m, n, dma, sigma,
                                    sum_mode, res[3] ? 0 : 2, (uint8_t*)(b + offs_ord[gi]),
                                    (double*)(b + offs_ms[gi]), (uint32_t*)(b + offs_ns[gi]))))
            return rc;
        const uint64_t lo = los[gi];
        CK(cudaMemcpyAsync(order + lo * n, b + offs_ord[gi], m * n, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(makespan + lo, b + offs_ms[gi], m * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        if (n_sims)
            CK(cudaMemcpyAsync(n_sims + lo, b + offs_ns[gi], m * sizeof(uint32_t), cudaMemcpyDeviceToHost,
                               c->stream));
    }
    for (int gi = 0; gi < G; ++gi) {
        DevCtx* c = dl.v[gi];
        if (!ms_[gi]) continue;
        CK(cudaSetDevice(c->dev));
        if ((rc = finish(c, c->stream))) return rc;
    }
    return 0;
}

int osim_heuristic_batch_dev(const double* d_durs, const uint8_t* d_id_rank, uint64_t B, int n,
                             int dma, double sigma, int sum_mode, int fast, uint8_t* d_order,
                             double* d_makespan, uint32_t* d_n_sims, void* stream) {
    int rc = check_common(n, dma, sigma);
    if (rc) return rc;
    DevList dl;
    if ((rc = pick_devs(1, dl))) return rc;
    DevCtx* c = dl.v[0];
    std::lock_guard<std::mutex> lk(c->mu);
    return enqueue_heuristic(c, stream ? (cudaStream_t)stream : c->stream, d_durs, d_id_rank, B, n, dma,
                             sigma, sum_mode, fast, d_order, d_makespan, d_n_sims);
}

int osim_timeline(const double* durs, int n, int dma, double sigma, const uint8_t* order,
                  double* start, double* end, double* makespan, double* idle) {
    if (n > kMaxN) return osim_timeline_deps(durs, n, dma, sigma, order, nullptr, 0, start, end, makespan, idle);
    int rc = check_common(n, dma, sigma);
    if (rc) return rc;
    if ((rc = check_durs(durs, (uint64_t)n))) return rc;
    if (!order || !start || !end) return fail(OSIM_EINVAL, "NULL buffer");
    unsigned seen = 0;
    for (int j = 0; j < n; ++j) {
        if (order[j] >= n || ((seen >> order[j]) & 1u)) return fail(OSIM_EINVAL, "order is not a permutation");
        seen |= 1u << order[j];
    }
    DevList dl;
    if ((rc = pick_devs(1, dl))) return rc;
    DevCtx* c = dl.v[0];
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->dev));
    size_t off_o = align_up(3 * kMaxN * sizeof(double));
    size_t off_s = off_o + 256;
    size_t off_e = off_s + align_up(3 * kMaxN * sizeof(double));
    size_t off_r = off_e + align_up(3 * kMaxN * sizeof(double));
    void* base;
    if ((rc = scratch(c, off_r + 256, &base))) return rc;
    char* b = (char*)base;
    CK(cudaMemcpyAsync(b, durs, 3 * n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(b + off_o, order, n, cudaMemcpyHostToDevice, c->stream));
    if (dma == 2)
        k_timeline<2><<<1, 64, 0, c->stream>>>((double*)b, n, sigma, (uint8_t*)(b + off_o), (double*)(b + off_s),
                                               (double*)(b + off_e), (double*)(b + off_r), c->d_err);
    else
        k_timeline<1><<<1, 64, 0, c->stream>>>((double*)b, n, sigma, (uint8_t*)(b + off_o), (double*)(b + off_s),
                                               (double*)(b + off_e), (double*)(b + off_r), c->d_err);
    CK(cudaGetLastError());
    double res[4];
    CK(cudaMemcpyAsync(start, b + off_s, 3 * n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(end, b + off_e, 3 * n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(res, b + off_r, sizeof(res), cudaMemcpyDeviceToHost, c->stream));
    if ((rc = finish(c, c->stream))) return rc;
    if (makespan) *makespan = res[0];
    if (idle) { idle[0] = res[1]; idle[1] = res[2]; idle[2] = res[3]; }
    return 0;
}

// ---- row f1: NoReorder interleavings (workload.py:259-327) ---------------

static uint64_t multinomial_total(int T, int N) {  // (T*N)! / (N!)^T, exact
    uint64_t r = 1;
    int tot = 0;
    for (int w = 0; w < T; ++w)
        for (int k = 1; k <= N; ++k) {
            ++tot;
            r = r / (uint64_t)k * (uint64_t)tot + r % (uint64_t)k * (uint64_t)tot / (uint64_t)k;
        }
    return r;
}

int osim_interleavings(const double* durs, int T, int N, int dma, double sigma, uint64_t rank_lo,
                       uint64_t rank_hi, double threshold, int n_dev, osim_summary* out, uint64_t* below,
                       double* makespans) {
    if (T < 1 || N < 1 || T * N > kMaxN) return fail(OSIM_EINVAL, "T*N must be in [1, %d]", kMaxN);
    int rc = check_common(T * N, dma, sigma);
    if (rc) return rc;
    int fast = 0;
    if ((rc = scan_durs(durs, (uint64_t)(T * N), sigma, &fast))) return rc;
    if (!out) return fail(OSIM_EINVAL, "out is NULL");
    const uint64_t total = multinomial_total(T, N);
    if (rank_lo > rank_hi || rank_hi > total) return fail(OSIM_EINVAL, "rank range outside [0, %llu)",
                                                          (unsigned long long)total);
    DevList dl;
    if ((rc = pick_devs(n_dev, dl))) return rc;
    const int G = (int)dl.v.size();
    const uint64_t span = rank_hi - rank_lo;
    std::vector<osim_summary> res(G);
    std::vector<unsigned long long> bel(G, 0);
    std::vector<std::unique_lock<std::mutex>> locks;
    for (int gi = 0; gi < G; ++gi) {
        DevCtx* c = dl.v[gi];
        locks.emplace_back(c->mu);
        CK(cudaSetDevice(c->dev));
        const uint64_t lo = rank_lo + span * (uint64_t)gi / (uint64_t)G;
        const uint64_t hi = rank_lo + span * (uint64_t)(gi + 1) / (uint64_t)G;
        const int mp = max_parts_for(c);
        size_t off_parts = align_up(3 * kMaxN * sizeof(double));
        size_t off_sum = off_parts + align_up(mp * sizeof(Part));
        size_t off_bel = off_sum + align_up(sizeof(osim_summary));
        size_t off_ms = off_bel + 256;
        size_t bytes = off_ms + (makespans ? align_up((hi - lo) * sizeof(double)) : 0);
        void* base;
        if ((rc = scratch(c, bytes, &base))) return rc;
        char* b = (char*)base;
        CK(cudaMemcpyAsync(b, durs, 3 * T * N * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        double* d_ms = makespans ? (double*)(b + off_ms) : nullptr;
        int g = 0;
        if (hi > lo) {
            const uint64_t blocks = (hi - lo + kBlock - 1) / kBlock;
            if (dma == 2 && fast == 1) {
                // runs of kRun consecutive ranks share their common label prefix
                const int run = f1_run_len();
                const uint64_t rb = ((hi - lo + run - 1) / run + kBlock - 1) / kBlock;
                auto k = sigma_pow2(sigma) ? (T * N <= 15 ? k_interleave_pfx<true, true> : k_interleave_pfx<true, false>)
                                           : (T * N <= 15 ? k_interleave_pfx<false, true> : k_interleave_pfx<false, false>);
                g = grid_for(k, kBlock, 0, c, rb);
                if (g > mp) g = mp;
                k<<<g, kBlock, 0, c->stream>>>((double*)b, T, N, sigma, lo, hi, total, run, threshold,
                                               (Part*)(b + off_parts), d_ms, c->d_err);
            } else if (dma == 1 && fast == 1) {
                const int run = f1_run_len();
                const uint64_t rb = ((hi - lo + run - 1) / run + kBlock - 1) / kBlock;
                auto k = T * N <= 15 ? k_interleave_pfx1<true> : k_interleave_pfx1<false>;
                g = grid_for(k, kBlock, 0, c, rb);
                if (g > mp) g = mp;
                k<<<g, kBlock, 0, c->stream>>>((double*)b, T, N, lo, hi, total, run, threshold,
                                               (Part*)(b + off_parts), d_ms, c->d_err);
            } else if (dma == 2) {
                g = grid_for(k_interleave<2>, kBlock, 0, c, blocks);
                if (g > mp) g = mp;
                k_interleave<2><<<g, kBlock, 0, c->stream>>>((double*)b, T, N, sigma, lo, hi, total, threshold,
                                                             (Part*)(b + off_parts), d_ms, c->d_err);
            } else {
                g = grid_for(k_interleave<1>, kBlock, 0, c, blocks);
                if (g > mp) g = mp;
                k_interleave<1><<<g, kBlock, 0, c->stream>>>((double*)b, T, N, sigma, lo, hi, total, threshold,
                                                             (Part*)(b + off_parts), d_ms, c->d_err);
            }
        }
        k_final_reduce<<<1, kBlock, 0, c->stream>>>((Part*)(b + off_parts), g, (osim_summary*)(b + off_sum),
                                                    (unsigned long long*)(b + off_bel));
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(&res[gi], b + off_sum, sizeof(osim_summary), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(&bel[gi], b + off_bel, sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream));
        if (makespans && hi > lo)
            CK(cudaMemcpyAsync(makespans + (lo - rank_lo), d_ms, (hi - lo) * sizeof(double),
                               cudaMemcpyDeviceToHost, c->stream));
    }
    osim_summary acc;
    memset(&acc, 0, sizeof(acc));
    uint64_t nb = 0;
    for (int gi = 0; gi < G; ++gi) {
        DevCtx* c = dl.v[gi];
        CK(cudaSetDevice(c->dev));
        if ((rc = finish(c, c->stream))) return rc;
        merge_host(acc, res[gi]);
        nb += bel[gi];
    }
    *out = acc;
    if (below) *below = nb;
    return 0;
}

int osim_eval_sequences(const double* durs, int T, int N, int dma, double sigma, const uint8_t* labels,
                        uint64_t cnt, int n_dev, double* makespans, osim_summary* out) {
    if (T < 1 || N < 1 || T * N > kWideMaxN) return fail(OSIM_EINVAL, "T*N must be in [1, %d]", kWideMaxN);
    int rc = check_common(T * N, dma, sigma, kWideMaxN);
    if (rc) return rc;
    if ((rc = check_durs(durs, (uint64_t)(T * N)))) return rc;
    if (cnt && (!labels || !makespans)) return fail(OSIM_EINVAL, "NULL buffer");
    const int n = T * N;
    for (uint64_t i = 0; i < cnt; ++i) {  // each row: every worker exactly N times
        int c[kWideMaxN] = {0};
        for (int p = 0; p < n; ++p) {
            const int w = labels[i * n + p];
            if (w >= T || ++c[w] > N)
                return fail(OSIM_EINVAL, "row %llu is not an interleaving of %d workers x %d tasks",
                            (unsigned long long)i, T, N);
        }
    }
    DevList dl;
    if ((rc = pick_devs(n_dev, dl))) return rc;
    const int G = (int)dl.v.size();
    std::vector<osim_summary> res(G);
    std::vector<std::unique_lock<std::mutex>> locks;
    for (int gi = 0; gi < G; ++gi) {
        DevCtx* c = dl.v[gi];
        locks.emplace_back(c->mu);
        CK(cudaSetDevice(c->dev));
        const uint64_t lo = cnt * (uint64_t)gi / (uint64_t)G, hi = cnt * (uint64_t)(gi + 1) / (uint64_t)G;
        const uint64_t m = hi - lo;
        const int mp = max_parts_for(c);
        size_t off_parts = align_up(3 * kWideMaxN * sizeof(double));
        size_t off_sum = off_parts + align_up(mp * sizeof(Part));
        size_t off_ms = off_sum + align_up(sizeof(osim_summary));
        size_t off_l = off_ms + align_up(m * sizeof(double) + 8);
        size_t bytes = off_l + align_up(m * n + 8);
        void* base;
        if ((rc = scratch(c, bytes, &base))) return rc;
        char* b = (char*)base;
        CK(cudaMemcpyAsync(b, durs, 3 * n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        int g = 0;
        if (m) {
            CK(cudaMemcpyAsync(b + off_l, labels + lo * n, m * n, cudaMemcpyHostToDevice, c->stream));
            const uint64_t blocks = (m + kBlock - 1) / kBlock;
            if (n > kMaxN) {  // 17..64 tasks: the byte-FIFO general path
                const LaunchCfg cfg{c->sms, c->stream};
                g = wide_eval_labels_launch(dma, cfg, (double*)b, T, N, sigma, (uint8_t*)(b + off_l), m,
                                            (double*)(b + off_ms), (Part*)(b + off_parts), mp, c->d_err);
            } else if (dma == 2) {
                g = grid_for(k_eval_labels<2>, kBlock, 0, c, blocks);
                if (g > mp) g = mp;
                k_eval_labels<2><<<g, kBlock, 0, c->stream>>>((double*)b, T, N, sigma, (uint8_t*)(b + off_l), m,
                                                              (Part*)(b + off_parts), (double*)(b + off_ms), c->d_err);
            } else {
                g = grid_for(k_eval_labels<1>, kBlock, 0, c, blocks);
                if (g > mp) g = mp;
                k_eval_labels<1><<<g, kBlock, 0, c->stream>>>((double*)b, T, N, sigma, (uint8_t*)(b + off_l), m,
                                                              (Part*)(b + off_parts), (double*)(b + off_ms), c->d_err);
            }
        }
        k_final_reduce<<<1, kBlock, 0, c->stream>>>((Part*)(b + off_parts), g, (osim_summary*)(b + off_sum), nullptr);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(&res[gi], b + off_sum, sizeof(osim_summary), cudaMemcpyDeviceToHost, c->stream));
        if (m) CK(cudaMemcpyAsync(makespans + lo, b + off_ms, m * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    }
    osim_summary acc;
    memset(&acc, 0, sizeof(acc));
    for (int gi = 0; gi < G; ++gi) {
        DevCtx* c = dl.v[gi];
        CK(cudaSetDevice(c->dev));
        if ((rc = finish(c, c->stream))) return rc;
        res[gi].best_rank += cnt * (uint64_t)gi / (uint64_t)G;
        merge_host(acc, res[gi]);
    }
    if (out) *out = acc;
    return 0;
}

int osim_timeline_deps(const double* durs, int n, int dma, double sigma, const uint8_t* order, const int8_t* dep,
                       int waves, double* start, double* end, double* makespan, double* idle) {
    int rc = check_common(n, dma, sigma, kWideMaxN);
    if (rc) return rc;
    if ((rc = check_durs(durs, (uint64_t)n))) return rc;
    if (!order || !start || !end) return fail(OSIM_EINVAL, "NULL buffer");
    uint64_t seen = 0;
    for (int j = 0; j < n; ++j) {
        if (order[j] >= n || ((seen >> order[j]) & 1ull)) return fail(OSIM_EINVAL, "order is not a permutation");
        seen |= 1ull << order[j];
    }
    if (dep)
        for (int t = 0; t < n; ++t)
            if (dep[t] >= n || dep[t] == t) return fail(OSIM_EINVAL, "bad dependency of task %d", t);
    DevList dl;
    if ((rc = pick_devs(1, dl))) return rc;
    DevCtx* c = dl.v[0];
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->dev));
    size_t off_o = align_up(3 * kWideMaxN * sizeof(double));
    size_t off_dp = off_o + 256;
    size_t off_s = off_dp + 256;
    size_t off_e = off_s + align_up(3 * kWideMaxN * sizeof(double));
    size_t off_r = off_e + align_up(3 * kWideMaxN * sizeof(double));
    void* base;
    if ((rc = scratch(c, off_r + 256, &base))) return rc;
    char* b = (char*)base;
    CK(cudaMemcpyAsync(b, durs, 3 * n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(b + off_o, order, n, cudaMemcpyHostToDevice, c->stream));
    if (dep) CK(cudaMemcpyAsync(b + off_dp, dep, n, cudaMemcpyHostToDevice, c->stream));
    const int8_t* d_dep = dep ? (const int8_t*)(b + off_dp) : nullptr;
    if (n > kMaxN)  // 17..64 tasks: the byte-FIFO general path
        wide_timeline_launch(dma, c->stream, (double*)b, n, sigma, (uint8_t*)(b + off_o), d_dep, waves,
                             (double*)(b + off_s), (double*)(b + off_e), (double*)(b + off_r), c->d_err);
    else if (dma == 2)
        k_timeline_dep<2><<<1, 64, 0, c->stream>>>((double*)b, n, sigma, (uint8_t*)(b + off_o), d_dep, waves,
                                                   (double*)(b + off_s), (double*)(b + off_e), (double*)(b + off_r),
                                                   c->d_err);
    else
        k_timeline_dep<1><<<1, 64, 0, c->stream>>>((double*)b, n, sigma, (uint8_t*)(b + off_o), d_dep, waves,
                                                   (double*)(b + off_s), (double*)(b + off_e), (double*)(b + off_r),
                                                   c->d_err);
    CK(cudaGetLastError());
    double res4[4];
    CK(cudaMemcpyAsync(start, b + off_s, 3 * n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(end, b + off_e, 3 * n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(res4, b + off_r, sizeof(res4), cudaMemcpyDeviceToHost, c->stream));
    if ((rc = finish(c, c->stream))) return rc;
    if (makespan) *makespan = res4[0];
    if (idle) { idle[0] = res4[1]; idle[1] = res4[2]; idle[2] = res4[3]; }
    return 0;
}

// ---- row f4: micro-step tick oracle (_micro.py, oracle.py:60-95) ----------

static long long micro_max_ticks(const double* durs, int n, double sigma, double dt) {
    double work = 0.0;  // every command runs at rate >= sigma: ticks <= total / (dt * sigma) + commands
    for (int i = 0; i < 3 * n; ++i) work += durs[i] > 0.0 ? durs[i] : 0.0;
    const double ticks = work / (dt * sigma) + 3.0 * n + 16.0;
    return ticks > 9.0e18 ? (long long)9.0e18 : (long long)ticks;
}

int osim_micro(const double* durs, int n, int dma, double sigma, double dt, uint64_t rank_lo, uint64_t rank_hi,
               int n_dev, double* makespans) {
    int rc = check_common(n, dma, sigma);
    if (rc) return rc;
    if (!(dt > 0.0)) return fail(OSIM_EINVAL, "dt must be positive");
    if ((rc = check_durs_micro(durs, (uint64_t)n))) return rc;
    if (!makespans && rank_hi > rank_lo) return fail(OSIM_EINVAL, "makespans is NULL");
    if (rank_lo > rank_hi || rank_hi > factorial(n)) return fail(OSIM_EINVAL, "bad rank range");
    const long long mt = micro_max_ticks(durs, n, sigma, dt);
    if ((double)mt * (double)(rank_hi - rank_lo) > 5e13)
        return fail(OSIM_EINVAL, "dt too small for this sweep (%lld ticks per ordering)", mt);
    DevList dl;
    if ((rc = pick_devs(n_dev, dl))) return rc;
    const int G = (int)dl.v.size();
    const uint64_t span = rank_hi - rank_lo;
    std::vector<std::unique_lock<std::mutex>> locks;
    for (int gi = 0; gi < G; ++gi) {
        DevCtx* c = dl.v[gi];
        locks.emplace_back(c->mu);
        CK(cudaSetDevice(c->dev));
        const uint64_t lo = rank_lo + span * (uint64_t)gi / (uint64_t)G;
        const uint64_t hi = rank_lo + span * (uint64_t)(gi + 1) / (uint64_t)G;
        if (hi <= lo) continue;
        size_t off_ms = align_up(3 * kMaxN * sizeof(double));
        void* base;
        if ((rc = scratch(c, off_ms + align_up((hi - lo) * sizeof(double)), &base))) return rc;
        char* b = (char*)base;
        CK(cudaMemcpyAsync(b, durs, 3 * n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        const unsigned blocks = (unsigned)((hi - lo + kBlock - 1) / kBlock);
        if (dma == 2)
            k_micro<2><<<blocks, kBlock, 0, c->stream>>>((double*)b, n, sigma, dt, lo, hi, mt, (double*)(b + off_ms),
                                                         c->d_err);
        else
            k_micro<1><<<blocks, kBlock, 0, c->stream>>>((double*)b, n, sigma, dt, lo, hi, mt, (double*)(b + off_ms),
                                                         c->d_err);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(makespans + (lo - rank_lo), b + off_ms, (hi - lo) * sizeof(double), cudaMemcpyDeviceToHost,
                           c->stream));
    }
    for (int gi = 0; gi < G; ++gi) {
        DevCtx* c = dl.v[gi];
        CK(cudaSetDevice(c->dev));
        if ((rc = finish(c, c->stream))) return rc;
    }
    return 0;
}

int osim_micro_timeline(const double* durs, int n, int dma, double sigma, double dt, const uint8_t* order,
                        double* start, double* end, double* makespan) {
    int rc = check_common(n, dma, sigma);
    if (rc) return rc;
    if (!(dt > 0.0)) return fail(OSIM_EINVAL, "dt must be positive");
    if ((rc = check_durs_micro(durs, (uint64_t)n))) return rc;
    if (!order || !start || !end) return fail(OSIM_EINVAL, "NULL buffer");
    unsigned seen = 0;
    for (int j = 0; j < n; ++j) {
        if (order[j] >= n || ((seen >> order[j]) & 1u)) return fail(OSIM_EINVAL, "order is not a permutation");
        seen |= 1u << order[j];
    }
    const long long mt = micro_max_ticks(durs, n, sigma, dt);
    if (mt > 4000000000ll) return fail(OSIM_EINVAL, "dt too small (%lld ticks)", mt);
    DevList dl;
    if ((rc = pick_devs(1, dl))) return rc;
    DevCtx* c = dl.v[0];
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->dev));
    size_t off_o = align_up(3 * kMaxN * sizeof(double));
    size_t off_s = off_o + 256;
    size_t off_e = off_s + align_up(3 * kMaxN * sizeof(double));
    size_t off_r = off_e + align_up(3 * kMaxN * sizeof(double));
    void* base;
    if ((rc = scratch(c, off_r + 256, &base))) return rc;
    char* b = (char*)base;
    CK(cudaMemcpyAsync(b, durs, 3 * n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(b + off_o, order, n, cudaMemcpyHostToDevice, c->stream));
    if (dma == 2)
        k_micro_timeline<2><<<1, 64, 0, c->stream>>>((double*)b, n, sigma, dt, (uint8_t*)(b + off_o), mt,
                                                     (double*)(b + off_s), (double*)(b + off_e), (double*)(b + off_r),
                                                     c->d_err);
    else
        k_micro_timeline<1><<<1, 64, 0, c->stream>>>((double*)b, n, sigma, dt, (uint8_t*)(b + off_o), mt,
                                                     (double*)(b + off_s), (double*)(b + off_e), (double*)(b + off_r),
                                                     c->d_err);
    CK(cudaGetLastError());
    double r0;
    CK(cudaMemcpyAsync(start, b + off_s, 3 * n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(end, b + off_e, 3 * n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(&r0, b + off_r, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    if ((rc = finish(c, c->stream))) return rc;
    if (makespan) *makespan = r0;
    return 0;
}

// ---- row f3: proxy-thread scenario harness (workload.py:197-256) ----------

int osim_harness_batch(const double* durs, const uint8_t* id_rank, uint64_t S, int T, int N, int dma, double sigma,
                       int sum_mode, int n_dev, double* makespan, uint8_t* n_groups, uint8_t* tg_sizes,
                       double* start, double* end) {
    if (T < 1 || N < 1 || T * N > kWideMaxN) return fail(OSIM_EINVAL, "T*N must be in [1, %d]", kWideMaxN);
    const int n = T * N;
    int rc = check_common(n, dma, sigma, kWideMaxN);
    if (rc) return rc;
    if ((rc = check_durs(durs, S * (uint64_t)n))) return rc;
    if (S && (!id_rank || !makespan || !n_groups)) return fail(OSIM_EINVAL, "NULL buffer");
    if ((rc = check_id_ranks(id_rank, S, n))) return rc;
    DevList dl;
    if ((rc = pick_devs(n_dev, dl))) return rc;
    const int G = (int)dl.v.size();
    std::vector<std::unique_lock<std::mutex>> locks;
    for (int gi = 0; gi < G; ++gi) {
        DevCtx* c = dl.v[gi];
        locks.emplace_back(c->mu);
        CK(cudaSetDevice(c->dev));
        const uint64_t lo = S * (uint64_t)gi / (uint64_t)G, hi = S * (uint64_t)(gi + 1) / (uint64_t)G;
        const uint64_t m = hi - lo;
        if (!m) continue;
        const bool tl = start && end;
        size_t off_r = align_up(m * n * 3 * sizeof(double));
        size_t off_ms = off_r + align_up(m * n);
        size_t off_ng = off_ms + align_up(m * sizeof(double));
        size_t off_sz = off_ng + align_up(m);
        size_t off_st = off_sz + align_up(m * n);
        size_t off_en = off_st + (tl ? align_up(m * n * 3 * sizeof(double)) : 0);
        size_t bytes = off_en + (tl ? align_up(m * n * 3 * sizeof(double)) : 0);
        void* base;
        if ((rc = scratch(c, bytes, &base))) return rc;
        char* b = (char*)base;
        CK(cudaMemcpyAsync(b, durs + lo * n * 3, m * n * 3 * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(b + off_r, id_rank + lo * n, m * n, cudaMemcpyHostToDevice, c->stream));
        // entries past a scenario's n_groups are zero (the kernels write the first n_groups)
        CK(cudaMemsetAsync(b + off_sz, 0, m * n, c->stream));
        const unsigned blocks = (unsigned)((m + 127) / 128);
        double* d_st = tl ? (double*)(b + off_st) : nullptr;
        double* d_en = tl ? (double*)(b + off_en) : nullptr;
        if (n > kMaxN)  // more than 16 tasks: WideSim FIFOs (osim_wide.cuh)
            wide_harness_launch(dma, c->stream, (double*)b, (uint8_t*)(b + off_r), m, T, N, sigma, sum_mode,
                                (double*)(b + off_ms), (uint8_t*)(b + off_ng), (uint8_t*)(b + off_sz), d_st, d_en,
                                c->d_err);
        else if (dma == 2)
            k_harness<2><<<blocks, 128, 0, c->stream>>>((double*)b, (uint8_t*)(b + off_r), m, T, N, sigma, sum_mode,
                                                        (double*)(b + off_ms), (uint8_t*)(b + off_ng),
                                                        (uint8_t*)(b + off_sz), d_st, d_en, c->d_err);
        else
            k_harness<1><<<blocks, 128, 0, c->stream>>>((double*)b, (uint8_t*)(b + off_r), m, T, N, sigma, sum_mode,
                                                        (double*)(b + off_ms), (uint8_t*)(b + off_ng),
                                                        (uint8_t*)(b + off_sz), d_st, d_en, c->d_err);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(makespan + lo, b + off_ms, m * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(n_groups + lo, b + off_ng, m, cudaMemcpyDeviceToHost, c->stream));
        if (tg_sizes) CK(cudaMemcpyAsync(tg_sizes + lo * n, b + off_sz, m * n, cudaMemcpyDeviceToHost, c->stream));
        if (tl) {
            CK(cudaMemcpyAsync(start + lo * n * 3, d_st, m * n * 3 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
            CK(cudaMemcpyAsync(end + lo * n * 3, d_en, m * n * 3 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        }
    }
    for (int gi = 0; gi < G; ++gi) {
        DevCtx* c = dl.v[gi];
        CK(cudaSetDevice(c->dev));
        if ((rc = finish(c, c->stream))) {
            if (rc == OSIM_ESTALL) return fail(OSIM_ESTALL, "harness stalled with tasks remaining");
            return rc;
        }
    }
    return 0;
}

int osim_selftest_div(uint64_t samples, uint64_t seed, uint64_t* mismatches) {
    DevList dl;
    int rc = pick_devs(1, dl);
    if (rc) return rc;
    DevCtx* c = dl.v[0];
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->dev));
    void* base;
    if ((rc = scratch(c, 256, &base))) return rc;
    CK(cudaMemsetAsync(base, 0, 8, c->stream));
    k_selftest_div<<<c->sms * 8, 256, 0, c->stream>>>(samples, seed, (unsigned long long*)base);
    CK(cudaGetLastError());
    unsigned long long h = 0;
    CK(cudaMemcpyAsync(&h, base, 8, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (mismatches) *mismatches = h;
    return 0;
}

int osim_selftest_div_mode(uint64_t samples, uint64_t seed, int mode, uint64_t* mismatches) {
    if (mode != 0 && mode != 1) return fail(OSIM_EINVAL, "mode must be 0 (random) or 1 (adversarial)");
    if (mode == 0) return osim_selftest_div(samples, seed, mismatches);
    DevList dl;
    int rc = pick_devs(1, dl);
    if (rc) return rc;
    DevCtx* c = dl.v[0];
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->dev));
    void* base;
    if ((rc = scratch(c, 256, &base))) return rc;
    CK(cudaMemsetAsync(base, 0, 8, c->stream));
    k_selftest_div_hard<<<c->sms * 8, 256, 0, c->stream>>>(samples, seed, (unsigned long long*)base);
    CK(cudaGetLastError());
    unsigned long long h = 0;
    CK(cudaMemcpyAsync(&h, base, 8, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (mismatches) *mismatches = h;
    return 0;
}

int osim_fp64_peak(double* tflops) {
    DevList dl;
    int rc = pick_devs(1, dl);
    if (rc) return rc;
    DevCtx* c = dl.v[0];
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->dev));
    void* base;
    if ((rc = scratch(c, 256, &base))) return rc;
    const int blocks = c->sms * 8, threads = 256, iters = 4096;
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    k_fp64_peak<<<blocks, threads, 0, c->stream>>>((double*)base, 64, 1.0000001, 1e-7);  // warm-up
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
        CK(cudaEventRecord(e0, c->stream));
        k_fp64_peak<<<blocks, threads, 0, c->stream>>>((double*)base, iters, 1.0000001, 1e-7);
        CK(cudaEventRecord(e1, c->stream));
        CK(cudaEventSynchronize(e1));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (ms < best) best = ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    const double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
    if (tflops) *tflops = flops / (best * 1e-3) / 1e12;
    return 0;
}

}  // extern "C"

// ---- groups of any size (osim_big.cuh): uint32 task ids -------------------
//
// The reference takes groups of any size (engine.py:252-263, oracle.py:127-135,
// heuristic.py:105-125, workload.py:197-304, oracle.py:60-95).  Up to 64
// tasks the uint8 entry points above run the register / byte-FIFO kernels;
// these entry points run BigSim with per-simulation workspaces in global
// memory for any n (ids below 2^31).

namespace {

int check_big(uint64_t n, int dma, double sigma) {
    if (n < 1) return fail(OSIM_EINVAL, "task group must be non-empty");
    if (n >= (1ull << 31)) return fail(OSIM_EINVAL, "n=%llu exceeds 2^31 - 1 tasks", (unsigned long long)n);
    if (dma != 1 && dma != 2) return fail(OSIM_EINVAL, "dma_engines must be 1 or 2, got %d", dma);
    if (!(sigma > 0.0 && sigma <= 1.0)) return fail(OSIM_EINVAL, "overlap_sigma must be in (0, 1]");
    return 0;
}

// rows of `width` uint32 values must each be a permutation of range(width)
int check_perm_rows(const uint32_t* v, uint64_t rows, uint64_t width, const char* what) {
    std::vector<uint64_t> stamp(width, ~0ull);
    for (uint64_t r = 0; r < rows; ++r)
        for (uint64_t j = 0; j < width; ++j) {
            const uint64_t x = v[r * width + j];
            if (x >= width || stamp[x] == r)
                return fail(OSIM_EINVAL, "%s row %llu is not a permutation of range(%llu)", what,
                            (unsigned long long)r, (unsigned long long)width);
            stamp[x] = r;
        }
    return 0;
}

// workspace budget of one big launch (per device), bytes
uint64_t big_budget() {
    static const uint64_t b = [] {
        const char* e = std::getenv("OSIM_BIG_WS_MB");  // testing / tuning only
        const long long mb = e ? std::atoll(e) : 0;
        return (uint64_t)(mb > 0 ? mb : 2048) << 20;
    }();
    return b;
}

// threads (a multiple of the block) whose per-thread workspaces of `per`
// bytes fit the budget, at most enough for `work` items and 8 CTAs per SM
int big_threads(const DevCtx* c, uint64_t per, uint64_t work, uint64_t* threads) {
    const uint64_t blk = (uint64_t)big_block();
    uint64_t t = big_budget() / (per ? per : 1);
    const uint64_t cap = (uint64_t)c->sms * 8 * blk;
    if (t > cap) t = cap;
    const uint64_t need = ((work + blk - 1) / blk) * blk;
    if (t > need) t = need;
    t = (t / blk) * blk;
    if (t == 0) {
        if (per > (16ull << 30)) return fail(OSIM_EINVAL, "workspace of %llu bytes per simulation is too large",
                                             (unsigned long long)per);
        t = blk;  // one CTA even above the budget
    }
    *threads = t;
    return 0;
}

}  // namespace

extern "C" {

int osim_timeline_u32(const double* durs, uint64_t n, int dma, double sigma, const uint32_t* order,
                      const int32_t* dep, int waves, double* start, double* end, double* makespan, double* idle) {
    int rc = check_big(n, dma, sigma);
    if (rc) return rc;
    if ((rc = check_durs(durs, n))) return rc;
    if (!order || !start || !end) return fail(OSIM_EINVAL, "NULL buffer");
    if ((rc = check_perm_rows(order, 1, n, "order"))) return rc;
    if (dep)
        for (uint64_t t = 0; t < n; ++t)
            if (dep[t] < -1 || dep[t] >= (int64_t)n || dep[t] == (int64_t)t)
                return fail(OSIM_EINVAL, "bad dependency of task %llu", (unsigned long long)t);
    DevList dl;
    if ((rc = pick_devs(1, dl))) return rc;
    DevCtx* c = dl.v[0];
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->dev));
    const size_t off_o = align_up(3 * n * sizeof(double));
    const size_t off_dp = off_o + align_up(n * sizeof(uint32_t));
    const size_t off_s = off_dp + align_up(n * sizeof(int32_t));
    const size_t off_e = off_s + align_up(3 * n * sizeof(double));
    const size_t off_r = off_e + align_up(3 * n * sizeof(double));
    const size_t off_ws = off_r + 256;
    void* base;
    if ((rc = scratch(c, off_ws + big_sim_bytes(n), &base))) return rc;
    char* b = (char*)base;
    CK(cudaMemcpyAsync(b, durs, 3 * n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(b + off_o, order, n * sizeof(uint32_t), cudaMemcpyHostToDevice, c->stream));
    if (dep) CK(cudaMemcpyAsync(b + off_dp, dep, n * sizeof(int32_t), cudaMemcpyHostToDevice, c->stream));
    big_timeline_launch(dma, c->stream, (double*)b, n, sigma, (uint32_t*)(b + off_o),
                        dep ? (int32_t*)(b + off_dp) : nullptr, waves, (uint8_t*)(b + off_ws), (double*)(b + off_s),
                        (double*)(b + off_e), (double*)(b + off_r), c->d_err);
    CK(cudaGetLastError());
    double res4[4];
    CK(cudaMemcpyAsync(start, b + off_s, 3 * n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(end, b + off_e, 3 * n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(res4, b + off_r, sizeof(res4), cudaMemcpyDeviceToHost, c->stream));
    if ((rc = finish(c, c->stream))) return rc;
    if (makespan) *makespan = res4[0];
    if (idle) { idle[0] = res4[1]; idle[1] = res4[2]; idle[2] = res4[3]; }
    return 0;
}

int osim_eval_perms_u32(const double* durs, uint64_t n, int dma, double sigma, const uint32_t* perms, uint64_t cnt,
                        int n_dev, double* makespans, osim_summary* out) {
    int rc = check_big(n, dma, sigma);
    if (rc) return rc;
    if ((rc = check_durs(durs, n))) return rc;
    if (cnt && (!perms || !makespans)) return fail(OSIM_EINVAL, "NULL buffer");
    if ((rc = check_perm_rows(perms, cnt, n, "perms"))) return rc;
    DevList dl;
    if ((rc = pick_devs(n_dev, dl))) return rc;
    const int G = (int)dl.v.size();
    std::vector<osim_summary> res(G);
    std::vector<std::unique_lock<std::mutex>> locks;
    const uint64_t wsb = big_sim_bytes(n);
    for (int gi = 0; gi < G; ++gi) {
        DevCtx* c = dl.v[gi];
        locks.emplace_back(c->mu);
        CK(cudaSetDevice(c->dev));
        const uint64_t lo = cnt * (uint64_t)gi / (uint64_t)G, hi = cnt * (uint64_t)(gi + 1) / (uint64_t)G;
        const uint64_t m = hi - lo;
        uint64_t threads = 0;
        if ((rc = big_threads(c, wsb, m, &threads))) return rc;
        const int grid = m ? (int)(threads / (uint64_t)big_block()) : 0;
        const size_t off_parts = align_up(3 * n * sizeof(double));
        const size_t off_sum = off_parts + align_up((grid + 1) * sizeof(Part));
        const size_t off_ms = off_sum + align_up(sizeof(osim_summary));
        const size_t off_p = off_ms + align_up(m * sizeof(double) + 8);
        const size_t off_ws = off_p + align_up(m * n * sizeof(uint32_t) + 8);
        void* base;
        if ((rc = scratch(c, off_ws + (m ? threads * wsb : 0), &base))) return rc;
        char* b = (char*)base;
        CK(cudaMemcpyAsync(b, durs, 3 * n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        Part* parts = (Part*)(b + off_parts);
        if (m) {
            CK(cudaMemcpyAsync(b + off_p, perms + lo * n, m * n * sizeof(uint32_t), cudaMemcpyHostToDevice,
                               c->stream));
            big_eval_perms_launch(dma, c->stream, grid, (double*)b, n, sigma, (uint32_t*)(b + off_p), m,
                                  (uint8_t*)(b + off_ws), wsb, (double*)(b + off_ms), parts, c->d_err);
        }
        k_final_reduce<<<1, kBlock, 0, c->stream>>>(parts, grid, (osim_summary*)(b + off_sum), nullptr);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(&res[gi], b + off_sum, sizeof(osim_summary), cudaMemcpyDeviceToHost, c->stream));
        if (m) CK(cudaMemcpyAsync(makespans + lo, b + off_ms, m * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    }
    osim_summary acc;
    memset(&acc, 0, sizeof(acc));
    for (int gi = 0; gi < G; ++gi) {
        DevCtx* c = dl.v[gi];
        CK(cudaSetDevice(c->dev));
        if ((rc = finish(c, c->stream))) return rc;
        res[gi].best_rank += cnt * (uint64_t)gi / (uint64_t)G;  // device-local indices -> list indices
        merge_host(acc, res[gi]);
    }
    if (out) *out = acc;
    return 0;
}

int osim_eval_sequences_u32(const double* durs, uint32_t T, uint32_t N, int dma, double sigma, const uint32_t* labels,
                            uint64_t cnt, int n_dev, double* makespans, osim_summary* out) {
    if (T < 1 || N < 1) return fail(OSIM_EINVAL, "T and N must be at least 1");
    const uint64_t n = (uint64_t)T * N;
    int rc = check_big(n, dma, sigma);
    if (rc) return rc;
    if ((rc = check_durs(durs, n))) return rc;
    if (cnt && (!labels || !makespans)) return fail(OSIM_EINVAL, "NULL buffer");
    {
        std::vector<uint32_t> cw(T);
        for (uint64_t i = 0; i < cnt; ++i) {  // each row: every worker exactly N times
            std::fill(cw.begin(), cw.end(), 0u);
            for (uint64_t p = 0; p < n; ++p) {
                const uint32_t w = labels[i * n + p];
                if (w >= T || ++cw[w] > N)
                    return fail(OSIM_EINVAL, "row %llu is not an interleaving of %u workers x %u tasks",
                                (unsigned long long)i, T, N);
            }
        }
    }
    std::vector<int32_t> dep(n);  // task (w, j) = w*N + j waits for (w, j-1) (workload.py:311-315)
    for (uint64_t t = 0; t < n; ++t) dep[t] = (t % N) ? (int32_t)(t - 1) : -1;
    DevList dl;
    if ((rc = pick_devs(n_dev, dl))) return rc;
    const int G = (int)dl.v.size();
    std::vector<osim_summary> res(G);
    std::vector<std::unique_lock<std::mutex>> locks;
    const uint64_t wsb = big_sim_bytes(n) + align_up((n + T) * sizeof(uint32_t));
    for (int gi = 0; gi < G; ++gi) {
        DevCtx* c = dl.v[gi];
        locks.emplace_back(c->mu);
        CK(cudaSetDevice(c->dev));
        const uint64_t lo = cnt * (uint64_t)gi / (uint64_t)G, hi = cnt * (uint64_t)(gi + 1) / (uint64_t)G;
        const uint64_t m = hi - lo;
        uint64_t threads = 0;
        if ((rc = big_threads(c, wsb, m, &threads))) return rc;
        const int grid = m ? (int)(threads / (uint64_t)big_block()) : 0;
        const size_t off_dep = align_up(3 * n * sizeof(double));
        const size_t off_parts = off_dep + align_up(n * sizeof(int32_t));
        const size_t off_sum = off_parts + align_up((grid + 1) * sizeof(Part));
        const size_t off_ms = off_sum + align_up(sizeof(osim_summary));
        const size_t off_l = off_ms + align_up(m * sizeof(double) + 8);
        const size_t off_ws = off_l + align_up(m * n * sizeof(uint32_t) + 8);
        void* base;
        if ((rc = scratch(c, off_ws + (m ? threads * wsb : 0), &base))) return rc;
        char* b = (char*)base;
        CK(cudaMemcpyAsync(b, durs, 3 * n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(b + off_dep, dep.data(), n * sizeof(int32_t), cudaMemcpyHostToDevice, c->stream));
        Part* parts = (Part*)(b + off_parts);
        if (m) {
            CK(cudaMemcpyAsync(b + off_l, labels + lo * n, m * n * sizeof(uint32_t), cudaMemcpyHostToDevice,
                               c->stream));
            big_eval_labels_launch(dma, c->stream, grid, (double*)b, T, N, sigma, (uint32_t*)(b + off_l), m,
                                   (int32_t*)(b + off_dep), (uint8_t*)(b + off_ws), wsb, (double*)(b + off_ms), parts,
                                   c->d_err);
        }
        k_final_reduce<<<1, kBlock, 0, c->stream>>>(parts, grid, (osim_summary*)(b + off_sum), nullptr);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(&res[gi], b + off_sum, sizeof(osim_summary), cudaMemcpyDeviceToHost, c->stream));
        if (m) CK(cudaMemcpyAsync(makespans + lo, b + off_ms, m * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    }
    osim_summary acc;
    memset(&acc, 0, sizeof(acc));
    for (int gi = 0; gi < G; ++gi) {
        DevCtx* c = dl.v[gi];
        CK(cudaSetDevice(c->dev));
        if ((rc = finish(c, c->stream))) return rc;
        res[gi].best_rank += cnt * (uint64_t)gi / (uint64_t)G;
        merge_host(acc, res[gi]);
    }
    if (out) *out = acc;
    return 0;
}

int osim_heuristic_batch_u32(const double* durs, const uint32_t* id_rank, uint64_t B, uint64_t n, int dma,
                             double sigma, int sum_mode, int n_dev, uint32_t* order, double* makespan,
                             uint32_t* n_sims) {
    int rc = check_big(n, dma, sigma);
    if (rc) return rc;
    if (n > 65535) return fail(OSIM_EINVAL, "n=%llu: the heuristic is limited to 65535 tasks per group",
                               (unsigned long long)n);
    if (B && (!durs || !id_rank || !order || !makespan)) return fail(OSIM_EINVAL, "NULL buffer");
    if ((rc = check_durs(durs, B * n))) return rc;
    if ((rc = check_perm_rows(id_rank, B, n, "id_rank"))) return rc;
    DevList dl;
    if ((rc = pick_devs(n_dev, dl))) return rc;
    const int G = (int)dl.v.size();
    std::vector<std::unique_lock<std::mutex>> locks;
    const uint64_t per_cta = big_heur_bytes_per_cta(n);
    for (int gi = 0; gi < G; ++gi) {
        DevCtx* c = dl.v[gi];
        locks.emplace_back(c->mu);
        CK(cudaSetDevice(c->dev));
        const uint64_t lo = B * (uint64_t)gi / (uint64_t)G, hi = B * (uint64_t)(gi + 1) / (uint64_t)G;
        const uint64_t m = hi - lo;
        if (!m) continue;
        uint64_t grid = big_budget() / per_cta;
        if (grid > (uint64_t)c->sms * 4) grid = (uint64_t)c->sms * 4;
        if (grid > m) grid = m;
        if (grid < 1) grid = 1;
        const size_t off_idr = align_up(m * 3 * n * sizeof(double));
        const size_t off_ord = off_idr + align_up(m * n * sizeof(uint32_t));
        const size_t off_ms = off_ord + align_up(m * n * sizeof(uint32_t));
        const size_t off_ns = off_ms + align_up(m * sizeof(double));
        const size_t off_ws = off_ns + align_up(m * sizeof(uint32_t));
        void* base;
        if ((rc = scratch(c, off_ws + grid * per_cta, &base))) return rc;
        char* b = (char*)base;
        CK(cudaMemcpyAsync(b, durs + lo * 3 * n, m * 3 * n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(b + off_idr, id_rank + lo * n, m * n * sizeof(uint32_t), cudaMemcpyHostToDevice,
                           c->stream));
        big_heuristic_launch(dma, c->stream, (int)grid, (double*)b, (uint32_t*)(b + off_idr), m, n, sigma, sum_mode,
                             (uint8_t*)(b + off_ws), (uint32_t*)(b + off_ord), (double*)(b + off_ms),
                             (uint32_t*)(b + off_ns), c->d_err);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(order + lo * n, b + off_ord, m * n * sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(makespan + lo, b + off_ms, m * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        if (n_sims)
            CK(cudaMemcpyAsync(n_sims + lo, b + off_ns, m * sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
    }
    for (int gi = 0; gi < G; ++gi) {
        DevCtx* c = dl.v[gi];
        CK(cudaSetDevice(c->dev));
        if ((rc = finish(c, c->stream))) return rc;
    }
    return 0;
}

int osim_harness_batch_u32(const double* durs, const uint32_t* id_rank, uint64_t S, uint32_t T, uint32_t N, int dma,
                           double sigma, int sum_mode, int n_dev, double* makespan, uint32_t* n_groups,
                           uint32_t* tg_sizes, double* start, double* end) {
    if (T < 1 || N < 1) return fail(OSIM_EINVAL, "T and N must be at least 1");
    const uint64_t n = (uint64_t)T * N;
    int rc = check_big(n, dma, sigma);
    if (rc) return rc;
    if (T > 65535) return fail(OSIM_EINVAL, "T=%u: at most 65535 workers", T);
    if ((rc = check_durs(durs, S * n))) return rc;
    if (S && (!id_rank || !makespan || !n_groups)) return fail(OSIM_EINVAL, "NULL buffer");
    if ((rc = check_perm_rows(id_rank, S, n, "id_rank"))) return rc;
    DevList dl;
    if ((rc = pick_devs(n_dev, dl))) return rc;
    const int G = (int)dl.v.size();
    std::vector<std::unique_lock<std::mutex>> locks;
    const uint64_t per = big_harness_bytes_per_thread(T, N);
    for (int gi = 0; gi < G; ++gi) {
        DevCtx* c = dl.v[gi];
        locks.emplace_back(c->mu);
        CK(cudaSetDevice(c->dev));
        const uint64_t lo = S * (uint64_t)gi / (uint64_t)G, hi = S * (uint64_t)(gi + 1) / (uint64_t)G;
        const uint64_t m = hi - lo;
        if (!m) continue;
        uint64_t threads = 0;
        if ((rc = big_threads(c, per, m, &threads))) return rc;
        const int grid = (int)(threads / (uint64_t)big_block());
        const bool tl = start && end;
        const size_t off_r = align_up(m * n * 3 * sizeof(double));
        const size_t off_ms = off_r + align_up(m * n * sizeof(uint32_t));
        const size_t off_ng = off_ms + align_up(m * sizeof(double));
        const size_t off_sz = off_ng + align_up(m * sizeof(uint32_t));
        const size_t off_st = off_sz + align_up(m * n * sizeof(uint32_t));
        const size_t off_en = off_st + (tl ? align_up(m * n * 3 * sizeof(double)) : 0);
        const size_t off_ws = off_en + (tl ? align_up(m * n * 3 * sizeof(double)) : 0);
        void* base;
        if ((rc = scratch(c, off_ws + threads * per, &base))) return rc;
        char* b = (char*)base;
        CK(cudaMemcpyAsync(b, durs + lo * n * 3, m * n * 3 * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(b + off_r, id_rank + lo * n, m * n * sizeof(uint32_t), cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemsetAsync(b + off_sz, 0, m * n * sizeof(uint32_t), c->stream));
        double* d_st = tl ? (double*)(b + off_st) : nullptr;
        double* d_en = tl ? (double*)(b + off_en) : nullptr;
        big_harness_launch(dma, c->stream, grid, (double*)b, (uint32_t*)(b + off_r), m, T, N, sigma, sum_mode,
                           (uint8_t*)(b + off_ws), (double*)(b + off_ms), (uint32_t*)(b + off_ng),
                           (uint32_t*)(b + off_sz), d_st, d_en, c->d_err);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(makespan + lo, b + off_ms, m * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(n_groups + lo, b + off_ng, m * sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
        if (tg_sizes)
            CK(cudaMemcpyAsync(tg_sizes + lo * n, b + off_sz, m * n * sizeof(uint32_t), cudaMemcpyDeviceToHost,
                               c->stream));
        if (tl) {
            CK(cudaMemcpyAsync(start + lo * n * 3, d_st, m * n * 3 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
            CK(cudaMemcpyAsync(end + lo * n * 3, d_en, m * n * 3 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        }
    }
    for (int gi = 0; gi < G; ++gi) {
        DevCtx* c = dl.v[gi];
        CK(cudaSetDevice(c->dev));
        if ((rc = finish(c, c->stream))) {
            if (rc == OSIM_ESTALL) return fail(OSIM_ESTALL, "harness stalled with tasks remaining");
            return rc;
        }
    }
    return 0;
}

int osim_micro_timeline_u32(const double* durs, uint64_t n, int dma, double sigma, double dt, const uint32_t* order,
                            double* start, double* end, double* makespan) {
    int rc = check_big(n, dma, sigma);
    if (rc) return rc;
    if (!(dt > 0.0)) return fail(OSIM_EINVAL, "dt must be positive");
    if ((rc = check_durs_micro(durs, n))) return rc;
    if (!order || !start || !end) return fail(OSIM_EINVAL, "NULL buffer");
    if ((rc = check_perm_rows(order, 1, n, "order"))) return rc;
    double work = 0.0;  // every command runs at rate >= sigma: ticks <= total / (dt * sigma) + commands
    for (uint64_t i = 0; i < 3 * n; ++i) work += durs[i] > 0.0 ? durs[i] : 0.0;
    const double tk = work / (dt * sigma) + 3.0 * (double)n + 16.0;
    if (tk > 4.0e9) return fail(OSIM_EINVAL, "dt too small (%.3g ticks)", tk);
    const long long mt = (long long)tk;
    DevList dl;
    if ((rc = pick_devs(1, dl))) return rc;
    DevCtx* c = dl.v[0];
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->dev));
    const size_t off_o = align_up(3 * n * sizeof(double));
    const size_t off_s = off_o + align_up(n * sizeof(uint32_t));
    const size_t off_e = off_s + align_up(3 * n * sizeof(double));
    const size_t off_r = off_e + align_up(3 * n * sizeof(double));
    void* base;
    if ((rc = scratch(c, off_r + 256, &base))) return rc;
    char* b = (char*)base;
    CK(cudaMemcpyAsync(b, durs, 3 * n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(b + off_o, order, n * sizeof(uint32_t), cudaMemcpyHostToDevice, c->stream));
    big_micro_timeline_launch(dma, c->stream, (double*)b, n, sigma, dt, (uint32_t*)(b + off_o), mt,
                              (double*)(b + off_s), (double*)(b + off_e), (double*)(b + off_r), c->d_err);
    CK(cudaGetLastError());
    double r0;
    CK(cudaMemcpyAsync(start, b + off_s, 3 * n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(end, b + off_e, 3 * n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(&r0, b + off_r, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    if ((rc = finish(c, c->stream))) return rc;
    if (makespan) *makespan = r0;
    return 0;
}

}  // extern "C"
