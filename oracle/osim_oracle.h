/*
 * osim_oracle.h -- CPU restatement of the reference simulator path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the parity checker for the
 * CUDA path (tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg).  It is never linked into, or called by, the
 * product library paper_1806_10113_b200/liboffsim_b200.so.
 *
 * Parity pinned: every function is checked bit-for-bit against fixtures
 * generated from the unmodified reference (tests/golden/make_golden.py,
 * Python 3.12.3 in the build container).
 */
#ifndef OSIM_ORACLE_H
#define OSIM_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    double best;
    uint64_t best_rank;
    double worst;
    double sum;
    double sum_log;
    uint64_t count;
} oracle_summary;

/* engine.simulate (engine.py:252-263) for one ordered task group.
 * durs: [n_tasks][3] (t_htd, t_k, t_dth) per task index.
 * order: [n_order] task indices (the submission order).
 * dep: nullable [n_tasks] prerequisite task index or -1 (engine.py:168-171).
 * start/end: nullable [n_tasks][3]; -1 marks a null stage (no command).
 * Returns 0, -1 (bad input / unresolvable), -5 (stalled, engine.py:239-241). */
int oracle_simulate(const double* durs, int n_tasks, int dma, double sigma,
                    const int* order, int n_order, const int* dep,
                    double* start, double* end, double* makespan,
                    double* idle /*[3] HtD,K,DtH nullable*/, double* k_end,
                    int* n_steps);

/* Instrumentation: summed (steps, running-command-steps, sigma-rate
 * transfer-steps) over ranks lo, lo+stride, ... < hi. */
int oracle_op_stats(const double* durs, int n, int dma, double sigma, uint64_t lo, uint64_t hi,
                    uint64_t stride, int64_t* out);

/* Calling thread's (S, R, O, simulations) totals over oracle_simulate. */
void oracle_stats_reset(void);
void oracle_stats_get(int64_t* out);

/* Lehmer unrank: rank -> lexicographic permutation of range(n)
 * (itertools.permutations order, oracle.py:125). */
void oracle_unrank(uint64_t rank, int n, int* perm);

/* exhaustive_search's simulate-and-reduce loop (oracle.py:132-135 +
 * make_report oracle.py:41-57) over ranks [lo, hi), on `threads` host
 * threads.  makespans nullable [hi-lo]. */
int oracle_exhaustive(const double* durs, int n, int dma, double sigma,
                      uint64_t lo, uint64_t hi, int threads,
                      oracle_summary* out, double* makespans);

/* Explicit permutation list (sampled mode, oracle.py:98-108,127-135). */
int oracle_eval_perms(const double* durs, int n, int dma, double sigma,
                      const uint8_t* perms, uint64_t cnt, int threads,
                      double* makespans, oracle_summary* out);

/* heuristic.reorder_batch (heuristic.py:105-125).  id_rank[i] = position
 * of task i in Python's sorted() order of ids.  sum_mode: 1 = CPython>=3.12
 * Neumaier builtin sum, 0 = naive left-to-right sum. */
int oracle_reorder(const double* durs, const uint8_t* id_rank, int n, int dma,
                   double sigma, int sum_mode, uint8_t* order,
                   double* makespan, uint32_t* n_sims);

/* Batched reorder over B independent groups on `threads` host threads. */
int oracle_reorder_batch(const double* durs, const uint8_t* id_rank,
                         uint64_t B, int n, int dma, double sigma,
                         int sum_mode, int threads, uint8_t* order,
                         double* makespan, uint32_t* n_sims);

/* workload.simulate_sequence (workload.py:277-304): deps gate, and on a
 * 1-DMA device the wave split into separate submits. */
int oracle_simulate_seq(const double* durs, int n_tasks, int dma, double sigma, const int* order, int n_order,
                        const int* dep, double* start, double* end, double* makespan, double* idle);
/* sorted(set(permutations(labels))) rank -> label sequence (workload.py:262-265). */
void oracle_unrank_labels(uint64_t rank, int T, int N, int* labels);
/* noreorder_distribution (workload.py:307-327) over label-sequence ranks
 * [lo, hi); durs [T][N][3], task (w, j) depends on (w, j-1). */
int oracle_interleavings(const double* durs, int T, int N, int dma, double sigma, uint64_t lo, uint64_t hi,
                         int threads, oracle_summary* out, double* makespans);
/* sampled mode: explicit label sequences labels[cnt][T*N]. */
int oracle_eval_sequences(const double* durs, int T, int N, int dma, double sigma, const uint8_t* labels,
                          uint64_t cnt, int threads, double* makespans, oracle_summary* out);

/* oracle.micro_simulate's core (_micro.py:19-143): fixed-dt tick loop over
 * the tasks in `order`; start/end by task index. */
int oracle_micro(const double* durs, int n, int dma, double sigma, double dt, const int* order, double* start,
                 double* end, double* makespan);

/* workload._run_heuristic_schedule (workload.py:197-256): proxy-thread
 * harness of one scenario; durs [T][N][3], id_rank [T*N] (sorted() order of
 * all task ids); tg_sizes nullable [T*N]. */
int oracle_harness(const double* durs, const uint8_t* id_rank, int T, int N, int dma, double sigma, int sum_mode,
                   double* makespan, int* n_groups, int* tg_sizes);

/* CPython builtin sum() of doubles (bltinmodule.c, 3.12 Neumaier / <=3.11
 * naive), exposed for the tests. */
double oracle_pysum(const double* x, int n, int sum_mode);

#ifdef __cplusplus
}
#endif
#endif
