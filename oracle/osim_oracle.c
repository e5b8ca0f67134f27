/*
 * osim_oracle.c -- CPU restatement of the reference simulator path.
 *
 * TEST INFRASTRUCTURE ONLY (see osim_oracle.h).  Only tests/,
 * __graft_entry__.smoke() and bench.py's CPU-baseline leg load this; the
 * product CUDA library never does.
 *
 * This is a deliberately literal restatement of the reference's
 * object-based algorithm (queues of command records, readiness checks,
 * per-step rate/dt/update/finalize) so that it can serve as the oracle the
 * fast, register-resident GPU formulation is checked against.  Citations
 * are /root/reference/pkg/src/offsim/<file>:<line>.
 *
 * Build with -O2 -ffp-contract=off (no FMA contraction, SSE2 doubles):
 * every arithmetic operation below is one IEEE-754 double operation in
 * the same order as CPython evaluates the reference expression.
 */
#include "osim_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define OR_MAXN 320 /* tasks per group (stack arrays); the big.json goldens go to 300 */
#define OR_MAXN8 256 /* entry points with uint8 task indices or id ranks */
#define K_HTD 0 /* engine.py:18-21 KINDS = (HtD, K, DtH) */
#define K_K 1
#define K_DTH 2
#define END_EPS 1e-9 /* engine.py:26 */

typedef struct {
    int task;
    int kind;
    double nd;    /* nominal_duration */
    double start; /* -1 until started */
    double end;
    double rw;    /* remaining_work fraction, engine.py:36 */
} or_cmd;

typedef struct {
    int dma;
    double sigma;
    double now;
    int n_lanes;
    int lane_kind_is_k[3]; /* lane order: 2-DMA {HtD, DtH, K}; 1-DMA {XFER, K} */
    int q[3][2 * OR_MAXN];
    int qlen[3];
    int head[3];
    int exec[3]; /* executing command index or -1 */
    unsigned done[OR_MAXN]; /* bit per kind, engine.py:131-136 */
    int pending[OR_MAXN];
    int finished[OR_MAXN];
    const int* dep;
    or_cmd cmd[3 * OR_MAXN];
    int n_cmd;
    /* op-count instrumentation: steps, running-command
     * steps, running transfer-steps at rate sigma != 1 */
    int64_t st_S, st_R, st_O;
} or_sim;

/* DeviceSim.__init__ (engine.py:93-111) */
static void sim_init(or_sim* s, int dma, double sigma, const int* dep, int n_tasks) {
    /* only the bookkeeping that is read before written is cleared: the
     * oracle also serves as the timed CPU baseline, so no 11 KB memset */
    for (int l = 0; l < 3; ++l) { s->qlen[l] = 0; s->head[l] = 0; }
    for (int t = 0; t < n_tasks; ++t) s->finished[t] = 0;
    s->n_cmd = 0;
    s->st_S = s->st_R = s->st_O = 0;
    s->dma = dma;
    s->sigma = sigma;
    s->now = 0.0;
    if (dma == 2) {
        /* dict order HtD, DtH, K (engine.py:98-102) */
        s->n_lanes = 3;
        s->lane_kind_is_k[0] = 0;
        s->lane_kind_is_k[1] = 0;
        s->lane_kind_is_k[2] = 1;
    } else {
        s->n_lanes = 2; /* {"XFER", K} (engine.py:104) */
        s->lane_kind_is_k[0] = 0;
        s->lane_kind_is_k[1] = 1;
    }
    for (int l = 0; l < 3; ++l) s->exec[l] = -1;
    s->dep = dep;
}

/* DeviceSim._xfer_queue (engine.py:158-161) */
static int xfer_lane(const or_sim* s, int kind) {
    if (s->dma == 2) return kind == K_HTD ? 0 : 1;
    return 0;
}
static int k_lane(const or_sim* s) { return s->dma == 2 ? 2 : 1; }

static void push(or_sim* s, int lane, int c) { s->q[lane][s->qlen[lane]++] = c; }

static int new_cmd(or_sim* s, int task, int kind, double nd) {
    or_cmd* c = &s->cmd[s->n_cmd];
    c->task = task;
    c->kind = kind;
    c->nd = nd;
    c->start = -1.0;
    c->end = -1.0;
    c->rw = 1.0;
    return s->n_cmd++;
}

/* DeviceSim.submit (engine.py:115-156) */
static int sim_submit(or_sim* s, const double* durs, const int* order, int n_order) {
    int group_dth[OR_MAXN];
    int n_dth = 0;
    for (int i = 0; i < n_order; ++i) {
        int t = order[i];
        double th = durs[3 * t + 0], tk = durs[3 * t + 1], td = durs[3 * t + 2];
        if (th <= 0 && tk <= 0 && td <= 0) return -1; /* :129-130 */
        unsigned done = 0;
        int count = 0;
        if (th <= 0) done |= 1u << K_HTD; /* :133-135 */
        if (tk <= 0) done |= 1u << K_K;
        if (td <= 0) done |= 1u << K_DTH;
        s->done[t] = done;
        if (th > 0) { push(s, xfer_lane(s, K_HTD), new_cmd(s, t, K_HTD, th)); count++; }
        if (tk > 0) { push(s, k_lane(s), new_cmd(s, t, K_K, tk)); count++; }
        if (td > 0) { group_dth[n_dth++] = new_cmd(s, t, K_DTH, td); count++; }
        s->pending[t] = count;
    }
    /* One-DMA launch order: every HtD of the group before its DtHs (:153-154) */
    for (int i = 0; i < n_dth; ++i) push(s, xfer_lane(s, K_DTH), group_dth[i]);
    return 0;
}

/* DeviceSim._ready (engine.py:168-178) */
static int sim_ready(const or_sim* s, const or_cmd* c) {
    if (s->dep) {
        int d = s->dep[c->task];
        if (d >= 0 && !s->finished[d]) return 0;
    }
    if (c->kind == K_K) return (s->done[c->task] >> K_HTD) & 1u;
    if (c->kind == K_DTH)
        return ((s->done[c->task] >> K_K) & 1u) && ((s->done[c->task] >> K_HTD) & 1u);
    return 1;
}

/* Python's max(left, 0.0): returns the first argument unless the second
 * compares greater (so max(-0.0, 0.0) is -0.0). */
static double py_max0(double left) { return (0.0 > left) ? 0.0 : left; }

/* DeviceSim.step (engine.py:182-232).  Returns the number of finalized
 * commands, or -1 when nothing runs (the `None` return). */
static int sim_step(or_sim* s) {
    for (int l = 0; l < s->n_lanes; ++l) { /* :188-194 */
        if (s->exec[l] < 0) {
            int h = s->head[l];
            if (h < s->qlen[l] && sim_ready(s, &s->cmd[s->q[l][h]])) {
                or_cmd* c = &s->cmd[s->q[l][h]];
                c->start = s->now;
                s->exec[l] = s->q[l][h];
            }
        }
    }
    int running[3], n_run = 0;
    for (int l = 0; l < s->n_lanes; ++l)
        if (s->exec[l] >= 0) running[n_run++] = s->exec[l]; /* :196 */
    if (n_run == 0) return -1;
    int any_h = 0, any_d = 0;
    for (int i = 0; i < n_run; ++i) {
        any_h |= s->cmd[running[i]].kind == K_HTD;
        any_d |= s->cmd[running[i]].kind == K_DTH;
    }
    int overlapped = s->dma == 2 && any_h && any_d; /* :200-204 */
    double rate[3];
    for (int i = 0; i < n_run; ++i) /* :207-208 */
        rate[i] = (overlapped && s->cmd[running[i]].kind != K_K) ? s->sigma : 1.0;
    /* :210  dt = min(rw * nd / rate) -- Python min keeps the first of equals */
    double dt = 0.0;
    for (int i = 0; i < n_run; ++i) {
        const or_cmd* c = &s->cmd[running[i]];
        double v = c->rw * c->nd / rate[i];
        if (i == 0 || v < dt) dt = v;
    }
    s->now += dt; /* :211 */
    s->st_S += 1;
    s->st_R += n_run;
    if (overlapped && s->sigma != 1.0)
        for (int i = 0; i < n_run; ++i) s->st_O += s->cmd[running[i]].kind != K_K;
    for (int i = 0; i < n_run; ++i) { /* :212-214 */
        or_cmd* c = &s->cmd[running[i]];
        double left = c->rw * c->nd - dt * rate[i];
        c->rw = py_max0(left) / c->nd;
    }
    static const int fin_order[3] = {K_HTD, K_DTH, K_K}; /* :24 */
    int n_fin = 0;
    for (int k = 0; k < 3; ++k) { /* :216-231 */
        for (int l = 0; l < s->n_lanes; ++l) {
            int ci = s->exec[l];
            if (ci < 0 || s->cmd[ci].kind != fin_order[k]) continue;
            or_cmd* c = &s->cmd[ci];
            if (c->rw * c->nd <= END_EPS) {
                c->rw = 0.0;
                c->end = s->now;
                s->exec[l] = -1;
                s->head[l] += 1;
                s->done[c->task] |= 1u << c->kind;
                if (--s->pending[c->task] == 0) s->finished[c->task] = 1;
                n_fin++;
            }
        }
    }
    return n_fin;
}

static int sim_drained(const or_sim* s) { /* :234-235 */
    for (int l = 0; l < s->n_lanes; ++l)
        if (s->head[l] < s->qlen[l]) return 0;
    return 1;
}

/* idle_report (engine.py:68-80): per kind, spans sorted by (start, end),
 * gaps accumulated left to right. */
static double idle_of_kind(const or_sim* s, int kind) {
    double st[3 * OR_MAXN], en[3 * OR_MAXN];
    int m = 0;
    for (int i = 0; i < s->n_cmd; ++i) {
        const or_cmd* c = &s->cmd[i];
        if (c->kind != kind || c->start < 0) continue;
        /* insertion sort on (start, end) */
        int j = m++;
        while (j > 0 && (st[j - 1] > c->start || (st[j - 1] == c->start && en[j - 1] > c->end))) {
            st[j] = st[j - 1];
            en[j] = en[j - 1];
            --j;
        }
        st[j] = c->start;
        en[j] = c->end;
    }
    double idle = 0.0;
    for (int i = 1; i < m; ++i)
        if (st[i] > en[i - 1]) idle += st[i] - en[i - 1];
    return idle;
}

/* thread-local instrumentation totals over every oracle_simulate call */
static __thread int64_t tl_stats[4];
void oracle_stats_reset(void) { tl_stats[0] = tl_stats[1] = tl_stats[2] = tl_stats[3] = 0; }
void oracle_stats_get(int64_t* out) { for (int i = 0; i < 4; ++i) out[i] = tl_stats[i]; }

int oracle_simulate(const double* durs, int n_tasks, int dma, double sigma,
                    const int* order, int n_order, const int* dep,
                    double* start, double* end, double* makespan, double* idle,
                    double* k_end, int* n_steps) {
    if (n_order < 1 || n_order > OR_MAXN || n_tasks > OR_MAXN) return -1; /* engine.py:258-259 */
    if (dma != 1 && dma != 2) return -1;
    or_sim s;
    sim_init(&s, dma, sigma, dep, n_tasks);
    if (sim_submit(&s, durs, order, n_order)) return -1;
    int steps = 0;
    while (!sim_drained(&s)) { /* run(), engine.py:237-241 */
        if (sim_step(&s) < 0) return -5;
        steps++;
    }
    tl_stats[0] += s.st_S;
    tl_stats[1] += s.st_R;
    tl_stats[2] += s.st_O;
    tl_stats[3] += 1;
    double ms = 0.0, ke = 0.0;
    int any = 0, anyk = 0;
    for (int i = 0; i < s.n_cmd; ++i) { /* timeline(), engine.py:246-249 */
        if (!any || s.cmd[i].end > ms) ms = s.cmd[i].end;
        any = 1;
        if (s.cmd[i].kind == K_K) { /* heuristic.py:46 max(K end, default=0.0) */
            if (!anyk || s.cmd[i].end > ke) ke = s.cmd[i].end;
            anyk = 1;
        }
    }
    if (makespan) *makespan = ms;
    if (k_end) *k_end = ke;
    if (n_steps) *n_steps = steps;
    if (idle) {
        idle[0] = idle_of_kind(&s, K_HTD);
        idle[1] = idle_of_kind(&s, K_K);
        idle[2] = idle_of_kind(&s, K_DTH);
    }
    if (start || end) {
        for (int t = 0; t < n_tasks * 3; ++t) {
            if (start) start[t] = -1.0;
            if (end) end[t] = -1.0;
        }
        for (int i = 0; i < s.n_cmd; ++i) {
            const or_cmd* c = &s.cmd[i];
            if (start) start[3 * c->task + c->kind] = c->start;
            if (end) end[3 * c->task + c->kind] = c->end;
        }
    }
    return 0;
}

/* Sum of (S, R, O) over ranks lo, lo+stride, ... < hi (instrumentation for
 * the roofline's algorithmic op count; not part of the reference). */
int oracle_op_stats(const double* durs, int n, int dma, double sigma, uint64_t lo, uint64_t hi,
                    uint64_t stride, int64_t* out) {
    int perm[OR_MAXN];
    out[0] = out[1] = out[2] = 0;
    if (stride < 1) stride = 1;
    for (uint64_t r = lo; r < hi; r += stride) {
        oracle_unrank(r, n, perm);
        or_sim s;
        sim_init(&s, dma, sigma, NULL, n);
        if (sim_submit(&s, durs, perm, n)) return -1;
        while (!sim_drained(&s))
            if (sim_step(&s) < 0) return -5;
        out[0] += s.st_S;
        out[1] += s.st_R;
        out[2] += s.st_O;
    }
    return 0;
}

/* itertools.permutations(range(n)) index == Lehmer rank (oracle.py:125) */
void oracle_unrank(uint64_t rank, int n, int* perm) {
    uint64_t fact[21];
    fact[0] = 1;
    for (int i = 1; i <= 20; ++i) fact[i] = fact[i - 1] * (uint64_t)i;
    int avail[OR_MAXN];
    for (int i = 0; i < n; ++i) avail[i] = i;
    int m = n;
    for (int i = 0; i < n; ++i) {
        uint64_t f = fact[n - 1 - i];
        int d = (int)(rank / f);
        rank %= f;
        perm[i] = avail[d];
        for (int j = d; j < m - 1; ++j) avail[j] = avail[j + 1];
        --m;
    }
}

/* make_report (oracle.py:41-57) reducer state: argmin keeps the first
 * index among ties (np.argmin), so `<` is strict. */
static void summary_init(oracle_summary* s) {
    s->best = 0.0;
    s->best_rank = 0;
    s->worst = 0.0;
    s->sum = 0.0;
    s->sum_log = 0.0;
    s->count = 0;
}
/* Neumaier-compensated accumulation so the oracle's mean/geomean are
 * accurate to a few ulps over 10^9 orderings (numpy's pairwise sum in the
 * reference is similarly accurate); the compensation terms live in the
 * per-thread job and are folded in before merging. */
typedef struct { double c_sum, c_log; } comp_t;
static void comp_add(double* s, double* c, double x) {
    double t = *s + x;
    if (fabs(*s) >= fabs(x)) *c += (*s - t) + x;
    else *c += (x - t) + *s;
    *s = t;
}
static void summary_add(oracle_summary* s, comp_t* cp, double ms, uint64_t rank) {
    if (s->count == 0 || ms < s->best) {
        s->best = ms;
        s->best_rank = rank;
    }
    if (s->count == 0 || ms > s->worst) s->worst = ms;
    comp_add(&s->sum, &cp->c_sum, ms);
    comp_add(&s->sum_log, &cp->c_log, log(ms));
    s->count++;
}
static void summary_merge(oracle_summary* a, const oracle_summary* b) {
    if (b->count == 0) return;
    if (a->count == 0) { *a = *b; return; }
    if (b->best < a->best) { a->best = b->best; a->best_rank = b->best_rank; }
    if (b->worst > a->worst) a->worst = b->worst;
    a->sum += b->sum;
    a->sum_log += b->sum_log;
    a->count += b->count;
}

typedef struct {
    const double* durs;
    int n, dma;
    double sigma;
    uint64_t lo, hi, base; /* rank range; base = global lo for makespans */
    const uint8_t* perms;  /* explicit list mode if non-null */
    double* makespans;
    oracle_summary sum;
    int err;
} ex_job;

static void* ex_worker(void* arg) {
    ex_job* j = (ex_job*)arg;
    summary_init(&j->sum);
    comp_t cp = {0.0, 0.0};
    int perm[OR_MAXN];
    for (uint64_t r = j->lo; r < j->hi; ++r) {
        if (j->perms) {
            for (int i = 0; i < j->n; ++i) perm[i] = j->perms[r * (uint64_t)j->n + i];
        } else {
            oracle_unrank(r, j->n, perm);
        }
        double ms;
        int rc = oracle_simulate(j->durs, j->n, j->dma, j->sigma, perm, j->n, NULL, NULL, NULL,
                                 &ms, NULL, NULL, NULL);
        if (rc) { j->err = rc; return NULL; }
        if (j->makespans) j->makespans[r - j->base] = ms;
        summary_add(&j->sum, &cp, ms, r);
    }
    j->sum.sum += cp.c_sum;
    j->sum.sum_log += cp.c_log;
    return NULL;
}

static int run_jobs(const double* durs, int n, int dma, double sigma, uint64_t lo, uint64_t hi,
                    const uint8_t* perms, int threads, double* makespans, oracle_summary* out) {
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    uint64_t total = hi - lo;
    if ((uint64_t)threads > total && total > 0) threads = (int)total;
    ex_job jobs[256];
    pthread_t tid[256];
    for (int t = 0; t < threads; ++t) {
        ex_job* j = &jobs[t];
        memset(j, 0, sizeof(*j));
        j->durs = durs; j->n = n; j->dma = dma; j->sigma = sigma;
        j->lo = lo + total * (uint64_t)t / (uint64_t)threads;
        j->hi = lo + total * (uint64_t)(t + 1) / (uint64_t)threads;
        j->base = lo; j->perms = perms; j->makespans = makespans;
    }
    if (threads == 1) {
        ex_worker(&jobs[0]);
    } else {
        for (int t = 0; t < threads; ++t) pthread_create(&tid[t], NULL, ex_worker, &jobs[t]);
        for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
    }
    oracle_summary acc;
    summary_init(&acc);
    for (int t = 0; t < threads; ++t) {
        if (jobs[t].err) return jobs[t].err;
        summary_merge(&acc, &jobs[t].sum);
    }
    if (out) *out = acc;
    return 0;
}

int oracle_exhaustive(const double* durs, int n, int dma, double sigma, uint64_t lo, uint64_t hi,
                      int threads, oracle_summary* out, double* makespans) {
    if (n < 1 || n > 20 || hi < lo) return -1; /* oracle.py:118-121 */
    return run_jobs(durs, n, dma, sigma, lo, hi, NULL, threads, makespans, out);
}

int oracle_eval_perms(const double* durs, int n, int dma, double sigma, const uint8_t* perms,
                      uint64_t cnt, int threads, double* makespans, oracle_summary* out) {
    if (n < 1 || n > OR_MAXN8) return -1;
    return run_jobs(durs, n, dma, sigma, 0, cnt, perms, threads, makespans, out);
}

/* CPython builtin sum over floats: 3.12+ Neumaier (bltinmodule.c
 * builtin_sum_impl), <=3.11 naive.  The int start value 0 is added to the
 * first element first (0 + x0). */
double oracle_pysum(const double* x, int n, int sum_mode) {
    if (n <= 0) return 0.0;
    double f = 0.0 + x[0];
    double c = 0.0;
    for (int i = 1; i < n; ++i) {
        if (sum_mode) {
            double t = f + x[i];
            if (fabs(f) >= fabs(x[i])) c += (f - t) + x[i];
            else c += (x[i] - t) + f;
            f = t;
        } else {
            f = f + x[i];
        }
    }
    if (sum_mode && c != 0.0 && isfinite(c)) f += c;
    return f;
}

/* ---- heuristic.py restatement ------------------------------------- */

typedef struct {
    const double* durs;
    const uint8_t* id_rank;
    int n, dma;
    double sigma;
    int sum_mode;
    uint32_t sims;
    int err;
} hctx;

static double h_sim(hctx* h, const int* seq, int len, double* k_end, double* idle_k) {
    double ms, idle[3], ke;
    int rc = oracle_simulate(h->durs, h->n, h->dma, h->sigma, seq, len, NULL, NULL, NULL, &ms,
                             idle, &ke, NULL);
    if (rc) h->err = rc;
    h->sims++;
    if (k_end) *k_end = ke;
    if (idle_k) *idle_k = idle[1];
    return ms;
}

/* select_first_task (heuristic.py:22-31): min over rt of
 * (-(t_k - t_htd), -t_dth, id); Python min keeps the first minimum. */
static int h_first(hctx* h, const int* rt, int m) {
    int best = -1;
    double b1 = 0, b2 = 0;
    for (int i = 0; i < m; ++i) {
        const double* d = h->durs + 3 * rt[i];
        double k1 = -(d[1] - d[0]);
        double k2 = -d[2];
        int less;
        if (best < 0) less = 1;
        else if (k1 < b1) less = 1;
        else if (b1 < k1) less = 0;
        else if (k2 < b2) less = 1;
        else if (b2 < k2) less = 0;
        else less = h->id_rank[rt[i]] < h->id_rank[best];
        if (less) { best = rt[i]; b1 = k1; b2 = k2; }
    }
    return best;
}

static void sort_by_id(const hctx* h, int* v, int m) { /* _by_id, heuristic.py:18-19 */
    for (int i = 1; i < m; ++i) {
        int x = v[i], j = i;
        while (j > 0 && h->id_rank[v[j - 1]] > h->id_rank[x]) { v[j] = v[j - 1]; --j; }
        v[j] = x;
    }
}

/* select_next_task (heuristic.py:52-78) with _completion_estimate (:34-49) */
static int h_next(hctx* h, const int* rt, int m, const int* ot, int k) {
    if (m == 1) return rt[0]; /* :67-68 */
    int cands[OR_MAXN];
    memcpy(cands, rt, sizeof(int) * m);
    sort_by_id(h, cands, m);
    int seq[OR_MAXN];
    memcpy(seq, ot, sizeof(int) * k);
    int best = -1;
    double be = 0, bi = 0;
    for (int ci = 0; ci < m; ++ci) {
        int cand = cands[ci];
        seq[k] = cand;
        double k_end, idle_k;
        double ms = h_sim(h, seq, k + 1, &k_end, &idle_k);
        /* rest = [r for r in rt if r is not cand], rt (input) order (:73) */
        double rk[OR_MAXN];
        int nr = 0;
        double tail = 0.0;
        for (int i = 0; i < m; ++i) {
            if (rt[i] == cand) continue;
            const double* d = h->durs + 3 * rt[i];
            rk[nr] = d[1];
            if (nr == 0 || d[2] < tail) tail = d[2]; /* min(... for r in rest) */
            nr++;
        }
        double rest_kernels = oracle_pysum(rk, nr, h->sum_mode);
        double bound = k_end + rest_kernels + tail; /* (k_end + rest) + tail */
        double est = (bound > ms) ? bound : ms;     /* max(makespan, bound) */
        int less;
        if (best < 0) less = 1;
        else if (est < be) less = 1;
        else if (be < est) less = 0;
        else if (idle_k < bi) less = 1;
        else if (bi < idle_k) less = 0;
        else less = h->id_rank[cand] < h->id_rank[best];
        if (less) { best = cand; be = est; bi = idle_k; }
    }
    return best;
}

/* select_last_tasks (heuristic.py:81-102) */
static void h_last(hctx* h, const int* rt, const int* ot, int k, int* o1, int* o2) {
    int ab[2] = {rt[0], rt[1]};
    sort_by_id(h, ab, 2);
    int a = ab[0], b = ab[1];
    int seq[OR_MAXN];
    memcpy(seq, ot, sizeof(int) * k);
    seq[k] = a; seq[k + 1] = b;
    double m_ab = h_sim(h, seq, k + 2, NULL, NULL);
    seq[k] = b; seq[k + 1] = a;
    double m_ba = h_sim(h, seq, k + 2, NULL, NULL);
    if (m_ab < m_ba) { *o1 = a; *o2 = b; return; }
    if (m_ba < m_ab) { *o1 = b; *o2 = a; return; }
    double dth_a = h->durs[3 * a + 2], dth_b = h->durs[3 * b + 2];
    if (dth_a <= dth_b) { *o1 = b; *o2 = a; } else { *o1 = a; *o2 = b; }
}

static void list_remove(int* v, int* m, int x) {
    for (int i = 0; i < *m; ++i)
        if (v[i] == x) {
            for (int j = i; j < *m - 1; ++j) v[j] = v[j + 1];
            (*m)--;
            return;
        }
}

/* reorder_batch (heuristic.py:105-125) */
int oracle_reorder(const double* durs, const uint8_t* id_rank, int n, int dma, double sigma,
                   int sum_mode, uint8_t* order, double* makespan, uint32_t* n_sims) {
    if (n < 1 || n > OR_MAXN8) return -1; /* :111-112 */
    hctx h = {durs, id_rank, n, dma, sigma, sum_mode, 0, 0};
    int ot[OR_MAXN] = {0}, k = 0;
    if (n == 1) {
        ot[k++] = 0;
    } else if (n == 2) {
        int rt[2] = {0, 1}, a, b;
        h_last(&h, rt, ot, 0, &a, &b);
        ot[k++] = a; ot[k++] = b;
    } else {
        int rt[OR_MAXN], m = n;
        for (int i = 0; i < n; ++i) rt[i] = i;
        int first = h_first(&h, rt, m);
        ot[k++] = first;
        list_remove(rt, &m, first);
        while (m > 2) {
            int nxt = h_next(&h, rt, m, ot, k);
            ot[k++] = nxt;
            list_remove(rt, &m, nxt);
        }
        int a, b;
        h_last(&h, rt, ot, k, &a, &b);
        ot[k++] = a; ot[k++] = b;
    }
    if (h.err) return h.err;
    uint32_t sims = h.sims;
    for (int i = 0; i < n; ++i) order[i] = (uint8_t)ot[i];
    if (makespan) {
        double ms;
        int rc = oracle_simulate(durs, n, dma, sigma, ot, n, NULL, NULL, NULL, &ms, NULL, NULL, NULL);
        if (rc) return rc;
        *makespan = ms;
    }
    if (n_sims) *n_sims = sims;
    return 0;
}

typedef struct {
    const double* durs;
    const uint8_t* id_rank;
    uint64_t lo, hi;
    int n, dma, sum_mode;
    double sigma;
    uint8_t* order;
    double* makespan;
    uint32_t* n_sims;
    int err;
} hb_job;

static void* hb_worker(void* arg) {
    hb_job* j = (hb_job*)arg;
    for (uint64_t b = j->lo; b < j->hi; ++b) {
        int rc = oracle_reorder(j->durs + b * 3 * (uint64_t)j->n, j->id_rank + b * (uint64_t)j->n,
                                j->n, j->dma, j->sigma, j->sum_mode, j->order + b * (uint64_t)j->n,
                                j->makespan ? j->makespan + b : NULL, j->n_sims ? j->n_sims + b : NULL);
        if (rc) { j->err = rc; return NULL; }
    }
    return NULL;
}

int oracle_reorder_batch(const double* durs, const uint8_t* id_rank, uint64_t B, int n, int dma,
                         double sigma, int sum_mode, int threads, uint8_t* order, double* makespan,
                         uint32_t* n_sims) {
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    if ((uint64_t)threads > B && B > 0) threads = (int)B;
    hb_job jobs[256];
    pthread_t tid[256];
    for (int t = 0; t < threads; ++t) {
        hb_job* j = &jobs[t];
        j->durs = durs; j->id_rank = id_rank; j->n = n; j->dma = dma; j->sum_mode = sum_mode;
        j->sigma = sigma; j->order = order; j->makespan = makespan; j->n_sims = n_sims; j->err = 0;
        j->lo = B * (uint64_t)t / (uint64_t)threads;
        j->hi = B * (uint64_t)(t + 1) / (uint64_t)threads;
    }
    if (threads == 1) hb_worker(&jobs[0]);
    else {
        for (int t = 0; t < threads; ++t) pthread_create(&tid[t], NULL, hb_worker, &jobs[t]);
        for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
    }
    for (int t = 0; t < threads; ++t)
        if (jobs[t].err) return jobs[t].err;
    return 0;
}


/* ---- workload.py restatement: NoReorder interleavings (row f1) ------ */

/* simulate_sequence (workload.py:277-304): 2-DMA or no deps -> one submit
 * with the deps gate; 1-DMA with deps -> a new wave (a separate submit)
 * whenever a task's prerequisite sits in the current wave. */
int oracle_simulate_seq(const double* durs, int n_tasks, int dma, double sigma, const int* order, int n_order,
                        const int* dep, double* start, double* end, double* makespan, double* idle) {
    if (n_order < 1 || n_order > OR_MAXN || n_tasks > OR_MAXN) return -1;
    if (dma != 2 && dep) {
        or_sim s;
        sim_init(&s, dma, sigma, dep, n_tasks);
        int wave[OR_MAXN], nw = 0;
        int in_wave[OR_MAXN];
        for (int t = 0; t < n_tasks; ++t) in_wave[t] = 0;
        for (int i = 0; i < n_order; ++i) {
            int t = order[i];
            int d = dep[t];
            if (d >= 0 && in_wave[d]) { /* workload.py:296-298 */
                if (sim_submit(&s, durs, wave, nw)) return -1;
                for (int j = 0; j < nw; ++j) in_wave[wave[j]] = 0;
                nw = 0;
            }
            wave[nw++] = t;
            in_wave[t] = 1;
        }
        if (nw && sim_submit(&s, durs, wave, nw)) return -1;
        while (!sim_drained(&s))
            if (sim_step(&s) < 0) return -5;
        double ms = 0.0;
        for (int i = 0; i < s.n_cmd; ++i)
            if (i == 0 || s.cmd[i].end > ms) ms = s.cmd[i].end;
        if (makespan) *makespan = ms;
        if (idle) {
            idle[0] = idle_of_kind(&s, K_HTD);
            idle[1] = idle_of_kind(&s, K_K);
            idle[2] = idle_of_kind(&s, K_DTH);
        }
        if (start || end) {
            for (int t = 0; t < n_tasks * 3; ++t) {
                if (start) start[t] = -1.0;
                if (end) end[t] = -1.0;
            }
            for (int i = 0; i < s.n_cmd; ++i) {
                const or_cmd* c = &s.cmd[i];
                if (start) start[3 * c->task + c->kind] = c->start;
                if (end) end[3 * c->task + c->kind] = c->end;
            }
        }
        return 0;
    }
    return oracle_simulate(durs, n_tasks, dma, sigma, order, n_order, dep, start, end, makespan, idle, NULL, NULL);
}

/* multinomial coefficient (sum c)! / prod c_i! for the remaining label counts */
static uint64_t multinom(const int* c, int T) {
    uint64_t r = 1;
    int tot = 0;
    for (int w = 0; w < T; ++w) {
        for (int k = 1; k <= c[w]; ++k) {
            ++tot;
            r = r * (uint64_t)tot / (uint64_t)k; /* exact: running binomial products */
        }
    }
    return r;
}

/* sorted(set(permutations(labels))) index -> label sequence (workload.py:262-265) */
void oracle_unrank_labels(uint64_t rank, int T, int N, int* labels) {
    int c[OR_MAXN];
    for (int w = 0; w < T; ++w) c[w] = N;
    for (int p = 0; p < T * N; ++p) {
        for (int w = 0; w < T; ++w) {
            if (!c[w]) continue;
            c[w]--;
            uint64_t m = multinom(c, T);
            if (rank < m) { labels[p] = w; break; }
            rank -= m;
            c[w]++;
        }
    }
}

/* labels -> task order and chain deps: task (w, j) is index w*N + j and
 * depends on (w, j-1) (noreorder_distribution, workload.py:310-326) */
static void labels_to_order(const int* labels, int T, int N, int* order, int* dep) {
    int cnt[OR_MAXN];
    for (int w = 0; w < T; ++w) cnt[w] = 0;
    for (int p = 0; p < T * N; ++p) order[p] = labels[p] * N + cnt[labels[p]]++;
    for (int w = 0; w < T; ++w)
        for (int j = 0; j < N; ++j) dep[w * N + j] = j ? w * N + j - 1 : -1;
}

typedef struct {
    const double* durs;
    int T, N, dma;
    double sigma;
    uint64_t lo, hi;
    const uint8_t* labels; /* explicit mode */
    double* makespans;
    oracle_summary sum;
    int err;
} il_job;

static void* il_worker(void* arg) {
    il_job* j = (il_job*)arg;
    summary_init(&j->sum);
    comp_t cp = {0.0, 0.0};
    int lab[OR_MAXN], order[OR_MAXN], dep[OR_MAXN];
    const int n = j->T * j->N;
    for (uint64_t r = j->lo; r < j->hi; ++r) {
        if (j->labels) for (int i = 0; i < n; ++i) lab[i] = j->labels[r * (uint64_t)n + i];
        else oracle_unrank_labels(r, j->T, j->N, lab);
        labels_to_order(lab, j->T, j->N, order, dep);
        double ms;
        int rc = oracle_simulate_seq(j->durs, n, j->dma, j->sigma, order, n, dep, NULL, NULL, &ms, NULL);
        if (rc) { j->err = rc; return NULL; }
        if (j->makespans) j->makespans[r] = ms;
        summary_add(&j->sum, &cp, ms, r);
    }
    j->sum.sum += cp.c_sum;
    j->sum.sum_log += cp.c_log;
    return NULL;
}

static int run_il(const double* durs, int T, int N, int dma, double sigma, uint64_t lo, uint64_t hi,
                  const uint8_t* labels, int threads, double* makespans, oracle_summary* out) {
    if (T < 1 || N < 1 || T * N > OR_MAXN) return -1;
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    uint64_t total = hi - lo;
    if ((uint64_t)threads > total && total > 0) threads = (int)total;
    il_job jobs[256];
    pthread_t tid[256];
    for (int t = 0; t < threads; ++t) {
        il_job* j = &jobs[t];
        memset(j, 0, sizeof(*j));
        j->durs = durs; j->T = T; j->N = N; j->dma = dma; j->sigma = sigma; j->labels = labels;
        j->lo = lo + total * (uint64_t)t / (uint64_t)threads;
        j->hi = lo + total * (uint64_t)(t + 1) / (uint64_t)threads;
        j->makespans = makespans ? makespans - lo : NULL;
    }
    if (threads == 1) il_worker(&jobs[0]);
    else {
        for (int t = 0; t < threads; ++t) pthread_create(&tid[t], NULL, il_worker, &jobs[t]);
        for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
    }
    oracle_summary acc;
    summary_init(&acc);
    for (int t = 0; t < threads; ++t) {
        if (jobs[t].err) return jobs[t].err;
        summary_merge(&acc, &jobs[t].sum);
    }
    if (out) *out = acc;
    return 0;
}

int oracle_interleavings(const double* durs, int T, int N, int dma, double sigma, uint64_t lo, uint64_t hi,
                         int threads, oracle_summary* out, double* makespans) {
    return run_il(durs, T, N, dma, sigma, lo, hi, NULL, threads, makespans, out);
}

int oracle_eval_sequences(const double* durs, int T, int N, int dma, double sigma, const uint8_t* labels,
                          uint64_t cnt, int threads, double* makespans, oracle_summary* out) {
    return run_il(durs, T, N, dma, sigma, 0, cnt, labels, threads, makespans, out);
}

/* ---- _micro.py restatement (row f4): fixed-dt tick loop ------------- */

/* _micro_core (_micro.py:19-143) over the tasks in `order`; start/end by
 * task index (-1 = no command). */
int oracle_micro(const double* durs, int n, int dma, double sigma, double dt, const int* order, double* start,
                 double* end, double* makespan) {
    if (n < 1 || n > OR_MAXN || !(dt > 0)) return -1;
    const double TOL = 1e-9; /* _micro.py:16 */
    int qh[OR_MAXN], qd[OR_MAXN], qk[OR_MAXN], nh = 0, nd = 0, nk = 0;
    double th[OR_MAXN], tk[OR_MAXN], td[OR_MAXN];
    for (int i = 0; i < n; ++i) { /* the sequence as micro_simulate sees it */
        const double* d = durs + 3 * order[i];
        th[i] = d[0]; tk[i] = d[1]; td[i] = d[2];
    }
    for (int i = 0; i < n; ++i) if (th[i] > 0.0) qh[nh++] = i;
    for (int i = 0; i < n; ++i) if (td[i] > 0.0) qd[nd++] = i;
    for (int i = 0; i < n; ++i) if (tk[i] > 0.0) qk[nk++] = i;
    double rem[3][OR_MAXN];
    int done[3][OR_MAXN];
    double st[3][OR_MAXN], en[3][OR_MAXN];
    for (int i = 0; i < n; ++i) {
        rem[0][i] = th[i]; rem[1][i] = tk[i]; rem[2][i] = td[i];
        done[0][i] = th[i] <= 0.0; done[1][i] = tk[i] <= 0.0; done[2][i] = td[i] <= 0.0;
        for (int k = 0; k < 3; ++k) st[k][i] = en[k][i] = -1.0;
    }
    int hh = 0, hd = 0, hk = 0;
    double t = 0.0, ms = 0.0;
    int64_t step = 0;
    for (;;) {
        int eh = -1, ed = -1, ek = -1;
        if (dma == 2) {
            if (hh < nh) eh = qh[hh];
            if (hd < nd) { int i = qd[hd]; if (done[1][i] && done[0][i]) ed = i; }
        } else {
            if (hh < nh) eh = qh[hh];
            else if (hd < nd) { int i = qd[hd]; if (done[1][i] && done[0][i]) ed = i; }
        }
        if (hk < nk) { int i = qk[hk]; if (done[0][i]) ek = i; }
        if (eh < 0 && ed < 0 && ek < 0) break;
        double rate = (dma == 2 && eh >= 0 && ed >= 0) ? sigma : 1.0;
        step += 1;
        double tick_end = (double)step * dt;
        if (eh >= 0) { if (st[0][eh] < 0.0) st[0][eh] = t; rem[0][eh] -= dt * rate; }
        if (ed >= 0) { if (st[2][ed] < 0.0) st[2][ed] = t; rem[2][ed] -= dt * rate; }
        if (ek >= 0) { if (st[1][ek] < 0.0) st[1][ek] = t; rem[1][ek] -= dt; }
        t = tick_end;
        if (eh >= 0 && rem[0][eh] <= TOL) { en[0][eh] = t; done[0][eh] = 1; hh++; ms = t; }
        if (ed >= 0 && rem[2][ed] <= TOL) { en[2][ed] = t; done[2][ed] = 1; hd++; ms = t; }
        if (ek >= 0 && rem[1][ek] <= TOL) { en[1][ek] = t; done[1][ek] = 1; hk++; ms = t; }
    }
    if (makespan) *makespan = ms;
    for (int i = 0; i < n; ++i) {
        const int task = order[i];
        for (int k = 0; k < 3; ++k) {
            if (start) start[3 * task + k] = st[k][i];
            if (end) end[3 * task + k] = en[k][i];
        }
    }
    return 0;
}

/* ---- workload.py restatement: proxy-thread harness (row f3) --------- */

/* _run_heuristic_schedule (workload.py:197-256) for one scenario: T workers
 * x N tasks, durs [T][N][3] (task (w, j) = index w*N + j), id_rank [T*N] =
 * position of each task id in sorted() order of all ids.  Returns the
 * timeline makespan, the number of groups and their sizes. */
int oracle_harness(const double* durs, const uint8_t* id_rank, int T, int N, int dma, double sigma, int sum_mode,
                   double* makespan, int* n_groups, int* tg_sizes) {
    const int n = T * N;
    if (T < 1 || N < 1 || n > OR_MAXN || T > 16) return -1;
    or_sim s;
    sim_init(&s, dma, sigma, NULL, n);
    int next_idx[16], avail[16], n_avail = 0, ng = 0;
    for (int w = 0; w < T; ++w) { next_idx[w] = 0; avail[n_avail++] = w; }
    int polling = 1, watched = -1;
    /* submit_group (workload.py:219-233) */
#define SUBMIT_GROUP()                                                                      \
    do {                                                                                    \
        int ws[16], m = 0;                                                                  \
        for (int w = 0; w < T; ++w)                                                         \
            for (int a = 0; a < n_avail; ++a)                                               \
                if (avail[a] == w) ws[m++] = w;                                             \
        int tg[16];                                                                         \
        double td[16 * 3] = {0};                                                            \
        uint8_t tr[16] = {0}, sub[16], order8[16];                                          \
        for (int i = 0; i < m; ++i) {                                                       \
            tg[i] = ws[i] * N + next_idx[ws[i]];                                            \
            next_idx[ws[i]]++;                                                              \
            for (int k = 0; k < 3; ++k) td[3 * i + k] = durs[3 * tg[i] + k];                \
        }                                                                                   \
        for (int i = 0; i < m; ++i) { /* ranks of the ids within the group */               \
            int r = 0;                                                                      \
            for (int j = 0; j < m; ++j) r += id_rank[tg[j]] < id_rank[tg[i]];               \
            tr[i] = (uint8_t)r;                                                             \
        }                                                                                   \
        n_avail = 0;                                                                        \
        if (oracle_reorder(td, tr, m, dma, sigma, sum_mode, order8, NULL, NULL)) return -1; \
        int ord[16];                                                                        \
        for (int i = 0; i < m; ++i) ord[i] = tg[order8[i]];                                 \
        (void)sub;                                                                          \
        int before = s.n_cmd;                                                               \
        if (sim_submit(&s, durs, ord, m)) return -1;                                        \
        if (tg_sizes) tg_sizes[ng] = m;                                                     \
        ng++;                                                                               \
        watched = -1;                                                                       \
        for (int c = before; c < s.n_cmd; ++c)                                              \
            if (s.cmd[c].kind == K_HTD) watched = c; /* htds[-1] */                         \
        polling = watched < 0;                                                              \
    } while (0)

    SUBMIT_GROUP();
    for (;;) {
        if (polling && n_avail) SUBMIT_GROUP();
        /* sim.step() with the finalized commands (engine.py:182-232) */
        int prev_exec[3];
        for (int l = 0; l < 3; ++l) prev_exec[l] = s.exec[l];
        (void)prev_exec;
        int before_done[3 * OR_MAXN];
        for (int c = 0; c < s.n_cmd; ++c) before_done[c] = s.cmd[c].end >= 0.0;
        int nf = sim_step(&s);
        if (nf < 0) {
            int remaining = 0;
            for (int w = 0; w < T; ++w) remaining |= next_idx[w] < N;
            if (remaining || !sim_drained(&s)) return -5; /* "harness stalled" */
            break;
        }
        /* finalized commands in _FINALIZE_ORDER (only sets/flags depend on them) */
        for (int c = 0; c < s.n_cmd; ++c) {
            if (before_done[c] || s.cmd[c].end < 0.0) continue;
            if (c == watched) polling = 1;
            const int t = s.cmd[c].task;
            if (s.finished[t]) {
                const int w = t / N, j = t % N;
                if (j + 1 < N) avail[n_avail++] = w;
            }
        }
    }
#undef SUBMIT_GROUP
    double ms = 0.0;
    for (int i = 0; i < s.n_cmd; ++i)
        if (i == 0 || s.cmd[i].end > ms) ms = s.cmd[i].end;
    if (makespan) *makespan = ms;
    if (n_groups) *n_groups = ng;
    return 0;
}
