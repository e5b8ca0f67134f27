/*
 * offsim_b200.h -- C ABI of liboffsim_b200.so, the B200 (sm_100a) hot path
 * of the temporal execution model of arXiv 1806.10113.
 *
 * The reference (`offsim`, /root/reference/pkg/src/offsim) is a pure-Python
 * package with no FFI; its public hot-path surface is three functions,
 * and each entry point below replaces the inner loop of one of them:
 *
 *   engine.simulate(tasks, profile)            engine.py:252-263
 *       -> osim_timeline           (one ordered group, full timeline)
 *   oracle.exhaustive_search(tasks, profile, cap, seed)   oracle.py:111-136
 *       -> osim_exhaustive         (every ordering: Lehmer ranks [lo, hi))
 *       -> osim_eval_perms         (sampled mode: explicit orderings,
 *                                   oracle.py:98-108,127-129)
 *       -> osim_exhaustive_batch   (many independent groups, one summary each)
 *   heuristic.reorder_batch(tg, profile)       heuristic.py:105-125
 *       -> osim_heuristic_batch    (Algorithm 1 over many groups)
 *
 * The summary replaces make_report's reductions (oracle.py:41-57):
 * best = ms.min(), best_rank = np.argmin(ms) (first of ties = lowest rank),
 * worst = ms.max(), sum -> mean, sum_log -> geomean = exp(sum_log / count).
 * The median needs the makespans (pass a `makespans` buffer).
 *
 * Durations are the resolved stage times (model.stage_times, model.py:139-160)
 * of each task as float64 (t_htd, t_k, t_dth) in ms, task-major [n][3];
 * a stage <= 0 is null (no command, engine.py:129-151).  `dma` is
 * DeviceProfile.dma_engines (1 or 2), `sigma` its overlap_sigma in (0, 1].
 * Orderings are task indices 0..n-1.  Group size: n <= 16 for the enumerated
 * spaces (osim_exhaustive*, osim_interleavings, osim_micro*, and every _dev
 * variant); n <= 64 for single orderings, explicit lists and scenarios
 * (osim_timeline, osim_timeline_deps, osim_eval_perms, osim_eval_sequences,
 * osim_heuristic_batch, osim_harness_batch), which above 16 tasks run on the
 * byte-FIFO general path.
 *
 * Conventions: every function returns 0 on success or a negative OSIM_E*
 * code; osim_last_error() gives a thread-local message.  Host buffers are
 * caller-owned, C-contiguous, used only during the call, never retained.
 * Device memory and streams are library-owned.  Calls are reentrant
 * (per-device mutex).  `_dev` variants take device pointers on the calling
 * thread's current library device, enqueue on `stream` (NULL = the
 * library's stream) and do not synchronize; they use the device's library
 * scratch (per-block partials, the last-block counter), so work enqueued by
 * _dev calls on one device must be ordered (one stream, or events between
 * streams) -- as in bench.py and dist.py.
 */
#ifndef OFFSIM_B200_H
#define OFFSIM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OSIM_OK 0
#define OSIM_EINVAL (-1)  /* ValueError / UnresolvableDuration in the reference */
#define OSIM_ENODEV (-2)  /* no CUDA device */
#define OSIM_ECUDA (-3)   /* CUDA runtime error */
#define OSIM_ENCCL (-4)   /* reserved: collective failure */
#define OSIM_ESTALL (-5)  /* "simulation stalled with commands pending", engine.py:239-241 */

/* make_report reduction state (48 bytes). */
typedef struct {
    double best;
    uint64_t best_rank; /* index of the first minimum within the evaluated set */
    double worst;
    double sum;
    double sum_log;
    uint64_t count;
} osim_summary;

/* Library version string. */
const char* osim_version(void);
/* Thread-local message for the last non-zero return on this thread. */
const char* osim_last_error(void);

/* Open up to `want_devices` CUDA devices (<= 0: all); *got = opened. */
int osim_init(int want_devices, int* got);
int osim_shutdown(void);
/* Select the library device used by this thread for n_dev <= 1 calls and
 * for the _dev variants (one process per GPU: pass LOCAL_RANK). */
int osim_set_device(int device);

/* exhaustive_search's simulate-and-reduce loop (oracle.py:123-135) over
 * lexicographic ranks [rank_lo, rank_hi) of range(n)'s permutations,
 * sharded over n_dev devices (<= 1: the current device).  `makespans`
 * (nullable) receives hi-lo values in rank order. */
int osim_exhaustive(const double* durs, int n, int dma, double sigma, uint64_t rank_lo,
                    uint64_t rank_hi, int n_dev, osim_summary* out, double* makespans);

/* Sampled mode: evaluate `cnt` explicit orderings perms[cnt][n]; best_rank
 * is the index in the list (np.argmin over the sample, oracle.py:47). */
int osim_eval_perms(const double* durs, int n, int dma, double sigma, const uint8_t* perms,
                    uint64_t cnt, int n_dev, double* makespans, osim_summary* out);

/* B independent groups durs[B][n][3], all n! orderings each; out[B]. */
int osim_exhaustive_batch(const double* durs, uint64_t B, int n, int dma, double sigma, int n_dev,
                          osim_summary* out);

/* reorder_batch (heuristic.py:105-125) for B groups.  id_rank[B][n]: the
 * position of each task in Python's sorted() order of the ids (the
 * tie-break of heuristic.py:18-19,29,74).  sum_mode: 1 = CPython >= 3.12
 * builtin sum (Neumaier), 0 = <= 3.11 naive (heuristic.py:47).
 * order[B][n] receives the chosen orderings, makespan[B] the simulated
 * makespan of each, n_sims[B] (nullable) the simulate() calls made. */
int osim_heuristic_batch(const double* durs, const uint8_t* id_rank, uint64_t B, int n, int dma,
                         double sigma, int sum_mode, int n_dev, uint8_t* order, double* makespan,
                         uint32_t* n_sims);

/* Order statistics of exhaustive_search without host lists (SURVEY.md 8(f)
 * row f2): the summary, *below = number of makespans strictly below
 * `threshold` (the `offsim permute` percentile numerator, cli.py:100-103;
 * -INFINITY counts none) and *median = np.median of the makespans of ranks
 * [rank_lo, rank_hi) (oracle.py:54; nullable).  The makespans stay in HBM
 * (8 bytes per ordering) and the median is an exact radix selection. */
int osim_exhaustive_stats(const double* durs, int n, int dma, double sigma, uint64_t rank_lo,
                          uint64_t rank_hi, double threshold, int n_dev, osim_summary* out,
                          uint64_t* below, double* median);

/* engine.simulate for one ordering: start/end[n][3] by task index
 * (-1 = null stage), makespan, idle[3] = idle_report (HtD, K, DtH). */
int osim_timeline(const double* durs, int n, int dma, double sigma, const uint8_t* order,
                  double* start, double* end, double* makespan, double* idle);

/* ---- NoReorder distribution (workload.py:259-327) */
/* T workers x N dependent tasks: durs[T*N][3] with task (w, j) at w*N + j
 * depending on (w, j-1).  Ranks index sorted(set(permutations(labels)))
 * (the worker-label sequences, workload.py:262-265); each sequence is
 * simulated as workload.simulate_sequence (deps gate; 1-DMA wave split,
 * :277-304).  below/threshold as in osim_exhaustive_stats; makespans
 * nullable [hi-lo]. */
int osim_interleavings(const double* durs, int T, int N, int dma, double sigma, uint64_t rank_lo,
                       uint64_t rank_hi, double threshold, int n_dev, osim_summary* out,
                       uint64_t* below, double* makespans);
/* Sampled mode: explicit worker-label rows labels[cnt][T*N]. */
int osim_eval_sequences(const double* durs, int T, int N, int dma, double sigma,
                        const uint8_t* labels, uint64_t cnt, int n_dev, double* makespans,
                        osim_summary* out);
/* engine.simulate(tasks, profile, deps) (waves = 0) or
 * workload.simulate_sequence (waves = 1): dep[n] = prerequisite task index
 * or -1 (nullable). */
int osim_timeline_deps(const double* durs, int n, int dma, double sigma, const uint8_t* order,
                       const int8_t* dep, int waves, double* start, double* end, double* makespan,
                       double* idle);

/* ---- proxy-thread scenario harness ----------- */
/* workload._run_heuristic_schedule (workload.py:197-256) for S independent
 * scenarios of T workers x N tasks: durs[S][T*N][3] (task (w, j) at w*N+j),
 * id_rank[S][T*N] = sorted() order of each scenario's task ids.  Outputs
 * makespan[S], n_groups[S], tg_sizes[S][T*N] (nullable; first n_groups entries, the rest 0),
 * start/end[S][T*N][3] (nullable; -1 = null stage). */
int osim_harness_batch(const double* durs, const uint8_t* id_rank, uint64_t S, int T, int N, int dma,
                       double sigma, int sum_mode, int n_dev, double* makespan, uint8_t* n_groups,
                       uint8_t* tg_sizes, double* start, double* end);

/* ---- micro-step validation oracle ------------- */
/* oracle.micro_simulate's fixed-dt tick loop (_micro.py:19-143,
 * oracle.py:60-95) for the orderings of ranks [lo, hi): makespans[hi-lo]. */
int osim_micro(const double* durs, int n, int dma, double sigma, double dt, uint64_t rank_lo,
               uint64_t rank_hi, int n_dev, double* makespans);
/* One ordering with its quantized timeline (start/end[n][3] by task, -1 = none). */
int osim_micro_timeline(const double* durs, int n, int dma, double sigma, double dt,
                        const uint8_t* order, double* start, double* end, double* makespan);

/* ---- device-resident variants (inputs already in HBM) ---------------- */
/* fast = 1 asserts every stage is non-null, every duration lies in
 * [2^-60, 2^22) ms and sigma >= 2^-60 (osim_fast_eligible()); for the
 * exhaustive and heuristic entry points fast = 2 asserts the same with null
 * (0) stages allowed (the null-stage fast simulator); 0 selects the general
 * path.  The host entry points choose the mode themselves. */
int osim_fast_eligible(const double* durs, uint64_t count /* tasks */, double sigma);
/* Suffix length L of the prefix-sharing kernels for n tasks (1..16): one
 * kernel call covers 512 prefixes x L! consecutive Lehmer ranks, and
 * osim_exhaustive_shard on the fast path gives shard r of W the calls
 * r, r + W, ...  (dist.shard_ranges mirrors it; OSIM_PFX_L may override it
 * for n in {8, 10, 12}, read once per process.) */
int osim_pfx_suffix_len(int n);

int osim_exhaustive_dev(const double* d_durs, int n, int dma, double sigma, uint64_t rank_lo,
                        uint64_t rank_hi, int fast, osim_summary* d_out, double* d_makespans,
                        void* stream);
/* Shard `shard` of `shards` of the whole space [0, n!) for multi-GPU strong
 * scaling (one call per rank; combine the summaries with the osim merge rules:
 * lowest best, ties to the lower best_rank).  On the fast path (fast = 1) the
 * shard is the interleaved set of 512-prefix calls shard, shard + shards, ...,
 * so every shard samples the whole rank space and the per-rank work evens
 * out; otherwise it is the contiguous range [shard*n!/shards,
 * (shard+1)*n!/shards).  Every ordering falls in exactly one shard.
 * Replaces, per rank, the enumeration loop of oracle.exhaustive_search
 * (/root/reference/pkg/src/offsim/oracle.py:124-135). */
int osim_exhaustive_shard_dev(const double* d_durs, int n, int dma, double sigma, int shard, int shards,
                              int fast, osim_summary* d_out, void* stream);
/* Host-buffer form of osim_exhaustive_shard_dev on the calling thread's
 * device (osim_set_device); chooses the path like osim_exhaustive.  The call
 * each rank of dist.exhaustive_summary_distributed makes. */
int osim_exhaustive_shard(const double* durs, int n, int dma, double sigma, int shard, int shards,
                          osim_summary* out);
/* As osim_exhaustive_dev plus the below-threshold count (d_below: one uint64). */
int osim_exhaustive_ex_dev(const double* d_durs, int n, int dma, double sigma, uint64_t rank_lo,
                           uint64_t rank_hi, int fast, double threshold, osim_summary* d_out,
                           uint64_t* d_below, double* d_makespans, void* stream);
/* One radix-selection pass over positive doubles in HBM: d_hist[2^digit_bits]
 * = histogram of the next digit_bits bits (MSB first) of the values whose top
 * prefix_bits bits equal `prefix` (digit_bits <= 11); 64-bit counts.  Ranks sum these
 * histograms (e.g. NCCL all_reduce) to select an order statistic of a
 * sharded makespan set. */
int osim_radix_hist_dev(const double* d_vals, uint64_t count, uint64_t prefix, int prefix_bits,
                        int digit_bits, uint64_t* d_hist, void* stream);
/* k-th smallest (0-based) of `count` non-negative doubles in HBM (no NaN, no
 * -0.0), by the same MSB-first radix selection with 64-bit bin counts that
 * osim_exhaustive_stats uses for np.median (oracle.py:54).  Waits for
 * `stream` (the producer of d_vals) first; synchronous. */
int osim_select_kth_dev(const double* d_vals, uint64_t count, uint64_t k, double* kth, void* stream);
int osim_exhaustive_batch_dev(const double* d_durs, uint64_t B, int n, int dma, double sigma,
                              int fast, osim_summary* d_out, void* stream);
int osim_heuristic_batch_dev(const double* d_durs, const uint8_t* d_id_rank, uint64_t B, int n,
                             int dma, double sigma, int sum_mode, int fast, uint8_t* d_order,
                             double* d_makespan, uint32_t* d_n_sims, void* stream);

/* ---- groups of any size (uint32 task ids) ------------------------------ */
/* The reference accepts task groups of any size; the uint8 entry points
 * above take up to 64 tasks.  These run the general path (osim_big.cuh:
 * FIFOs and done bits in per-simulation global-memory workspaces, IEEE
 * division, bit-identical to the reference) for any n < 2^31, with the same
 * argument meaning as their uint8 counterparts. */
/* engine.simulate / workload.simulate_sequence (engine.py:252-263,
 * workload.py:277-304): order[n], dep[n] (nullable; -1 = none), waves as in
 * osim_timeline_deps. */
int osim_timeline_u32(const double* durs, uint64_t n, int dma, double sigma, const uint32_t* order,
                      const int32_t* dep, int waves, double* start, double* end, double* makespan,
                      double* idle);
/* sampled exhaustive_search (oracle.py:127-135): perms[cnt][n]. */
int osim_eval_perms_u32(const double* durs, uint64_t n, int dma, double sigma, const uint32_t* perms,
                        uint64_t cnt, int n_dev, double* makespans, osim_summary* out);
/* NoReorder label sequences (workload.py:277-327): labels[cnt][T*N]. */
int osim_eval_sequences_u32(const double* durs, uint32_t T, uint32_t N, int dma, double sigma,
                            const uint32_t* labels, uint64_t cnt, int n_dev, double* makespans,
                            osim_summary* out);
/* reorder_batch (heuristic.py:105-125), n <= 65535: id_rank[B][n],
 * order[B][n]; one CTA per group, a greedy round's candidates spread over
 * its threads. */
int osim_heuristic_batch_u32(const double* durs, const uint32_t* id_rank, uint64_t B, uint64_t n, int dma,
                             double sigma, int sum_mode, int n_dev, uint32_t* order, double* makespan,
                             uint32_t* n_sims);
/* workload._run_heuristic_schedule (workload.py:197-256), T <= 65535. */
int osim_harness_batch_u32(const double* durs, const uint32_t* id_rank, uint64_t S, uint32_t T, uint32_t N,
                           int dma, double sigma, int sum_mode, int n_dev, double* makespan,
                           uint32_t* n_groups, uint32_t* tg_sizes, double* start, double* end);
/* oracle.micro_simulate (oracle.py:60-95). */
int osim_micro_timeline_u32(const double* durs, uint64_t n, int dma, double sigma, double dt,
                            const uint32_t* order, double* start, double* end, double* makespan);

/* ---- diagnostics ------------------------------------------------------ */
/* Compare the fast-path division with IEEE division on `samples` random
 * operand pairs drawn from the fast-path range; *mismatches = count. */
int osim_selftest_div(uint64_t samples, uint64_t seed, uint64_t* mismatches);
/* mode 0: as osim_selftest_div; mode 1: adversarial operands (mantissas on
 * rounding boundaries, quotients at binade edges, rounded products
 * y * (1 - 2^-k)) over the fast-path range of divisors [2^-60, 2^22). */
int osim_selftest_div_mode(uint64_t samples, uint64_t seed, int mode, uint64_t* mismatches);
/* Measured FP64 FMA-pipe throughput of the current device, TFLOP/s
 * (2 flops per DFMA). */
int osim_fp64_peak(double* tflops);

#ifdef __cplusplus
}
#endif
#endif
