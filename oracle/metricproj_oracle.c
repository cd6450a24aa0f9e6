/*
 * TEST INFRASTRUCTURE ONLY -- CPU oracle for the Dykstra triangle sweep.
 *
 * This file is a from-scratch C restatement of the reference solver's hot
 * path (arXiv 1901.10084 reference package `metricproj`).  It exists so that
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg have a checker and a CPU baseline that travel to the GPU box
 * (the Python/numba reference does not).  The product path never links or
 * calls it.
 *
 * Parity pin: the tests/golden fixtures were produced by the unmodified reference
 * (tests/golden/make_golden.py) and tests/test_oracle.py checks this oracle
 * against them bit for bit.
 *
 * Restated pieces (reference file:line):
 *   pair position ...................... _kernels.py:23-25, core.py:40-44
 *   tiled_rounds / diagonal_rounds ..... schedule.py:117-153, :94-114
 *   worker_of (pos+1) mod p ............. schedule.py:79-80
 *   metric_units_pass (cube order) ...... _kernels.py:60-132
 *   serial_metric_pass .................. _kernels.py:135-183
 *   pair_pass ........................... _kernels.py:186-220
 *   max_violation ....................... _kernels.py:28-57
 *   per-worker sparse duals + cursor .... core.py:218-256, solver.py:116-163
 *   barrier after every round ........... solver.py:150-151
 *   pair ranges w*m/p ................... solver.py:103-105
 *
 * Arithmetic is plain IEEE-754 double with no contraction (compile with
 * -ffp-contract=off), in exactly the association the reference uses.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define MPO_THETA_FLOOR 1e-15

static inline int64_t pidx(int64_t n, int64_t i, int64_t j) {
    return i * (n - 1) - i * (i - 1) / 2 + (j - i - 1);
}

/* ------------------------------------------------------------------ */
/* schedule                                                            */
/* ------------------------------------------------------------------ */

typedef struct {
    int64_t x, z;
} mpo_tile;

typedef struct {
    int64_t ntiles;
    int64_t first; /* offset into the flat tile array */
} mpo_round;

typedef struct {
    int64_t nrounds;
    mpo_round *rounds;
    int64_t ntiles;
    mpo_tile *tiles;
} mpo_schedule;

static int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }
static int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

/* Emit one anti-diagonal round starting at base (x, z), tiles offset by
 * (+c*b, -c*b) while the clipped tile is non-empty (schedule.py:124-130). */
static void emit_round(mpo_schedule *s, int64_t *cap_r, int64_t *cap_t,
                       int64_t x, int64_t z, int64_t b) {
    if (s->nrounds == *cap_r) {
        *cap_r = *cap_r ? 2 * *cap_r : 64;
        s->rounds = realloc(s->rounds, (size_t)*cap_r * sizeof(mpo_round));
    }
    mpo_round *r = &s->rounds[s->nrounds++];
    r->first = s->ntiles;
    r->ntiles = 0;
    for (int64_t c = 0; max64(x + c * b, 0) + 2 <= z - c * b; ++c) {
        if (s->ntiles == *cap_t) {
            *cap_t = *cap_t ? 2 * *cap_t : 256;
            s->tiles = realloc(s->tiles, (size_t)*cap_t * sizeof(mpo_tile));
        }
        s->tiles[s->ntiles].x = x + c * b;
        s->tiles[s->ntiles].z = z - c * b;
        s->ntiles++;
        r->ntiles++;
    }
}

/* The two double loops of schedule.py:132-152.  With b = 1 the tiles are
 * exactly the S_{i,k} sets of diagonal_rounds (schedule.py:94-114), which is
 * how Plan feeds "diagonal" to the kernel (solver.py:77,86-102). */
static void build_schedule(mpo_schedule *s, int64_t n, int64_t b) {
    int64_t cap_r = 0, cap_t = 0;
    memset(s, 0, sizeof(*s));
    for (int64_t z = n - 1; z >= 2; z -= b) emit_round(s, &cap_r, &cap_t, 1 - b, z, b);
    for (int64_t x = 1; x + 2 <= n - 1; x += b) emit_round(s, &cap_r, &cap_t, x, n - 1, b);
}

/* diagonal_rounds uses x = 0 for its first loop (schedule.py:106-109) while
 * tiled_rounds(b=1) uses x = 1 - b = 0: identical. */

/* ------------------------------------------------------------------ */
/* sparse dual arrays (one per worker)                                 */
/* ------------------------------------------------------------------ */

typedef struct {
    int64_t len, cap;
    int64_t *keys;
    double *vals;
} mpo_duals;

static void duals_push(mpo_duals *d, int64_t key, double val) {
    if (d->len == d->cap) {
        d->cap = d->cap ? 2 * d->cap : 1024;
        d->keys = realloc(d->keys, (size_t)d->cap * sizeof(int64_t));
        d->vals = realloc(d->vals, (size_t)d->cap * sizeof(double));
    }
    d->keys[d->len] = key;
    d->vals[d->len] = val;
    d->len++;
}

/* ------------------------------------------------------------------ */
/* solver state                                                        */
/* ------------------------------------------------------------------ */

typedef struct mpo_solver {
    int64_t n, m, b;
    int kind; /* 0 serial, 1 diagonal, 2 tiled */
    int workers;
    double eps;
    double *xv, *fv, *dflat, *winvx, *winvf, *pair_duals;
    mpo_schedule sched;
    mpo_duals *rd; /* read duals per worker (previous pass) */
    mpo_duals *wd; /* write duals per worker (this pass) */
    pthread_barrier_t barrier;
    /* per-pass worker results */
    double *wviol;
    int64_t *wsteps;
    int64_t round_limit; /* timing samples only: 0 = whole pass */
} mpo_solver;

/* One Dykstra step of a metric row; the three x positions and their W^-1
 * weights, in the reference's association (_kernels.py:115-129). */
static inline void metric_row(double *xv, const double *winvx, int64_t plus, int64_t m1,
                              int64_t m2, int64_t key, double eps, const mpo_duals *rd,
                              int64_t *cursor, mpo_duals *wd, double *viol) {
    double y_old = 0.0;
    if (*cursor < rd->len && rd->keys[*cursor] == key) {
        y_old = rd->vals[*cursor];
        (*cursor)++;
    }
    double d0 = xv[plus] - xv[m1] - xv[m2];
    if (d0 > *viol) *viol = d0;
    double s = winvx[plus] + winvx[m1] + winvx[m2];
    double delta = d0 + y_old * s / eps;
    double theta = delta > 0.0 ? eps * delta / s : 0.0;
    double coef = (y_old - theta) / eps;
    if (coef != 0.0) {
        xv[plus] += coef * winvx[plus];
        xv[m1] -= coef * winvx[m1];
        xv[m2] -= coef * winvx[m2];
    }
    if (theta > MPO_THETA_FLOOR) duals_push(wd, key, theta);
}

static inline void triplet(double *xv, const double *winvx, int64_t n, int64_t i, int64_t j,
                           int64_t k, double eps, const mpo_duals *rd, int64_t *cursor,
                           mpo_duals *wd, double *viol) {
    int64_t pij = pidx(n, i, j), pik = pidx(n, i, k), pjk = pidx(n, j, k);
    int64_t code = ((i * n + j) * n + k) * 3;
    /* kinds IJ, IK, JK: roles (plus, m1, m2) of _kernels.py:97-109 */
    metric_row(xv, winvx, pij, pik, pjk, code + 0, eps, rd, cursor, wd, viol);
    metric_row(xv, winvx, pik, pij, pjk, code + 1, eps, rd, cursor, wd, viol);
    metric_row(xv, winvx, pjk, pij, pik, code + 2, eps, rd, cursor, wd, viol);
}

/* Cube order inside a tile: j-chunks of width b, then k, j, i ascending
 * (_kernels.py:73-131, schedule.py:156-175). */
static int64_t tile_pass(mpo_solver *S, int64_t x, int64_t z, const mpo_duals *rd,
                         int64_t *cursor, mpo_duals *wd, double *viol) {
    const int64_t n = S->n, b = S->b;
    int64_t ilo = x > 0 ? x : 0, ihi = x + b - 1;
    int64_t klo = z - b + 1 > 0 ? z - b + 1 : 0;
    int64_t steps = 0;
    for (int64_t jb = x + 1; jb <= z - 1; jb += b) {
        int64_t je = min64(jb + b - 1, z - 1);
        int64_t jlo = jb > 1 ? jb : 1;
        for (int64_t k = klo; k <= z; ++k) {
            int64_t jtop = min64(je, k - 1);
            for (int64_t j = jlo; j <= jtop; ++j) {
                int64_t itop = min64(ihi, j - 1);
                for (int64_t i = ilo; i <= itop; ++i) {
                    triplet(S->xv, S->winvx, n, i, j, k, S->eps, rd, cursor, wd, viol);
                    steps += 3;
                }
            }
        }
    }
    return steps;
}

/* Both pair rows, upper then lower (_kernels.py:186-220). */
static int64_t pair_range(mpo_solver *S, int64_t lo, int64_t hi, double *viol) {
    double *xv = S->xv, *fv = S->fv;
    const double eps = S->eps;
    for (int64_t p = lo; p < hi; ++p) {
        double d = S->dflat[p];
        double s = S->winvx[p] + S->winvf[p];
        double y_old = S->pair_duals[2 * p];
        double d0 = xv[p] - fv[p] - d;
        if (d0 > *viol) *viol = d0;
        double delta = d0 + y_old * s / eps;
        double theta = delta > 0.0 ? eps * delta / s : 0.0;
        double coef = (y_old - theta) / eps;
        if (coef != 0.0) {
            xv[p] += coef * S->winvx[p];
            fv[p] -= coef * S->winvf[p];
        }
        S->pair_duals[2 * p] = theta > MPO_THETA_FLOOR ? theta : 0.0;
        y_old = S->pair_duals[2 * p + 1];
        d0 = d - xv[p] - fv[p];
        if (d0 > *viol) *viol = d0;
        delta = d0 + y_old * s / eps;
        theta = delta > 0.0 ? eps * delta / s : 0.0;
        coef = (y_old - theta) / eps;
        if (coef != 0.0) {
            xv[p] -= coef * S->winvx[p];
            fv[p] -= coef * S->winvf[p];
        }
        S->pair_duals[2 * p + 1] = theta > MPO_THETA_FLOOR ? theta : 0.0;
    }
    return 2 * (hi - lo);
}

typedef struct {
    mpo_solver *S;
    int w;
} mpo_job;

/* _worker_pass (solver.py:116-163): rounds with a barrier after each, then
 * the worker's contiguous pair range. */
static void *worker_main(void *arg) {
    mpo_job *job = (mpo_job *)arg;
    mpo_solver *S = job->S;
    const int w = job->w, p = S->workers;
    const mpo_duals *rd = &S->rd[w];
    mpo_duals *wd = &S->wd[w];
    int64_t cursor = 0, steps = 0;
    double viol = 0.0;
    wd->len = 0;
    if (S->kind == 0) {
        const int64_t n = S->n;
        for (int64_t i = 0; i < n - 2; ++i)
            for (int64_t j = i + 1; j < n - 1; ++j)
                for (int64_t k = j + 1; k < n; ++k) {
                    triplet(S->xv, S->winvx, n, i, j, k, S->eps, rd, &cursor, wd, &viol);
                    steps += 3;
                }
    } else {
        const int64_t nr = S->round_limit > 0 && S->round_limit < S->sched.nrounds
                               ? S->round_limit : S->sched.nrounds;
        for (int64_t r = 0; r < nr; ++r) {
            const mpo_round *R = &S->sched.rounds[r];
            for (int64_t pos = 0; pos < R->ntiles; ++pos) {
                if ((pos + 1) % p != w) continue;
                const mpo_tile *T = &S->sched.tiles[R->first + pos];
                steps += tile_pass(S, T->x, T->z, rd, &cursor, wd, &viol);
            }
            if (p > 1) pthread_barrier_wait(&S->barrier);
        }
    }
    int64_t lo = (int64_t)w * S->m / p, hi = (int64_t)(w + 1) * S->m / p;
    double pv = 0.0;
    if (S->round_limit <= 0) steps += pair_range(S, lo, hi, &pv);
    if (pv > viol) viol = pv;
    S->wviol[w] = viol;
    S->wsteps[w] = steps;
    return NULL;
}

/* ------------------------------------------------------------------ */
/* exported API (ctypes)                                               */
/* ------------------------------------------------------------------ */

mpo_solver *mpo_create(int64_t n, const double *d_flat, const double *reg_x,
                       const double *reg_f, double eps, int kind, int64_t b, int workers) {
    if (n < 3 || workers < 1 || b < 1 || kind < 0 || kind > 2) return NULL;
    if (kind == 0 && workers != 1) return NULL;
    mpo_solver *S = calloc(1, sizeof(mpo_solver));
    S->n = n;
    S->m = n * (n - 1) / 2;
    S->b = kind == 1 ? 1 : b;
    S->kind = kind;
    S->workers = workers;
    S->eps = eps;
    size_t bytes = (size_t)S->m * sizeof(double);
    S->xv = calloc(S->m, sizeof(double));
    S->fv = calloc(S->m, sizeof(double));
    S->dflat = malloc(bytes);
    S->winvx = malloc(bytes);
    S->winvf = malloc(bytes);
    S->pair_duals = calloc(2 * S->m, sizeof(double));
    memcpy(S->dflat, d_flat, bytes);
    for (int64_t p = 0; p < S->m; ++p) {
        S->winvx[p] = 1.0 / reg_x[p]; /* solver.py:173-174 */
        S->winvf[p] = 1.0 / reg_f[p];
    }
    if (kind != 0) build_schedule(&S->sched, n, S->b);
    S->rd = calloc(workers, sizeof(mpo_duals));
    S->wd = calloc(workers, sizeof(mpo_duals));
    S->wviol = calloc(workers, sizeof(double));
    S->wsteps = calloc(workers, sizeof(int64_t));
    if (workers > 1) pthread_barrier_init(&S->barrier, NULL, (unsigned)workers);
    return S;
}

void mpo_destroy(mpo_solver *S) {
    if (!S) return;
    for (int w = 0; w < S->workers; ++w) {
        free(S->rd[w].keys); free(S->rd[w].vals);
        free(S->wd[w].keys); free(S->wd[w].vals);
    }
    free(S->rd); free(S->wd); free(S->wviol); free(S->wsteps);
    free(S->xv); free(S->fv); free(S->dflat); free(S->winvx); free(S->winvf);
    free(S->pair_duals);
    free(S->sched.rounds); free(S->sched.tiles);
    if (S->workers > 1) pthread_barrier_destroy(&S->barrier);
    free(S);
}

/* State in/out in the reference's packed pair order (core.py:162-176). */
void mpo_set_state(mpo_solver *S, const double *xv, const double *fv) {
    memcpy(S->xv, xv, (size_t)S->m * sizeof(double));
    memcpy(S->fv, fv, (size_t)S->m * sizeof(double));
}

void mpo_get_state(const mpo_solver *S, double *xv, double *fv) {
    memcpy(xv, S->xv, (size_t)S->m * sizeof(double));
    memcpy(fv, S->fv, (size_t)S->m * sizeof(double));
}

void mpo_get_pair_duals(const mpo_solver *S, double *pd) {
    memcpy(pd, S->pair_duals, (size_t)(2 * S->m) * sizeof(double));
}

int64_t mpo_dual_count(const mpo_solver *S) {
    int64_t c = 0;
    for (int w = 0; w < S->workers; ++w) c += S->rd[w].len;
    return c;
}

/* Metric duals, workers concatenated in order (DualStore.items(),
 * core.py:243-247). */
void mpo_get_duals(const mpo_solver *S, int64_t *keys, double *vals) {
    int64_t off = 0;
    for (int w = 0; w < S->workers; ++w) {
        memcpy(keys + off, S->rd[w].keys, (size_t)S->rd[w].len * sizeof(int64_t));
        memcpy(vals + off, S->rd[w].vals, (size_t)S->rd[w].len * sizeof(double));
        off += S->rd[w].len;
    }
}

int64_t mpo_num_rounds(const mpo_solver *S) { return S->sched.nrounds; }
int64_t mpo_num_tiles(const mpo_solver *S) { return S->sched.ntiles; }

/* Flat schedule export: per round tile count, then (x, z) per tile. */
void mpo_get_schedule(const mpo_solver *S, int64_t *round_ntiles, int64_t *tiles_xz) {
    for (int64_t r = 0; r < S->sched.nrounds; ++r) round_ntiles[r] = S->sched.rounds[r].ntiles;
    for (int64_t t = 0; t < S->sched.ntiles; ++t) {
        tiles_xz[2 * t] = S->sched.tiles[t].x;
        tiles_xz[2 * t + 1] = S->sched.tiles[t].z;
    }
}

/* One full pass (run_pass, solver.py:166-210, minus the objective math,
 * which the Python wrapper does with numpy exactly as core.py does).
 * Returns the running max violation; *steps gets the step count. */
double mpo_run_pass(mpo_solver *S, int64_t *steps) {
    int p = S->workers;
    mpo_job *jobs = calloc(p, sizeof(mpo_job));
    pthread_t *th = calloc(p, sizeof(pthread_t));
    for (int w = 0; w < p; ++w) {
        jobs[w].S = S;
        jobs[w].w = w;
    }
    if (p == 1) {
        worker_main(&jobs[0]);
    } else {
        for (int w = 0; w < p; ++w) pthread_create(&th[w], NULL, worker_main, &jobs[w]);
        for (int w = 0; w < p; ++w) pthread_join(th[w], NULL);
    }
    double viol = 0.0;
    int64_t st = 0;
    for (int w = 0; w < p; ++w) {
        if (S->wviol[w] > viol) viol = S->wviol[w];
        st += S->wsteps[w];
        mpo_duals tmp = S->rd[w]; /* swap: this pass's writes are next pass's reads */
        S->rd[w] = S->wd[w];
        S->wd[w] = tmp;
    }
    free(jobs);
    free(th);
    if (steps) *steps = st;
    return viol;
}

/* Timing samples only (bench.py's P = 1 CPU row): later passes stop after the
 * first `limit` rounds of the tiled/diagonal schedule and skip the pair
 * phase, so `steps` counts exactly the metric rows visited.  0 restores
 * whole passes.  A limited pass leaves the solver mid-pass: not a result. */
void mpo_set_round_limit(mpo_solver *S, int64_t limit) { S->round_limit = limit; }

/* Exact violation scan (_kernels.py:28-57). */
double mpo_max_violation(const double *xv, const double *fv, const double *dflat, int64_t n) {
    double viol = 0.0;
    for (int64_t i = 0; i < n - 2; ++i)
        for (int64_t j = i + 1; j < n - 1; ++j) {
            int64_t pij = pidx(n, i, j);
            for (int64_t k = j + 1; k < n; ++k) {
                double xij = xv[pij], xik = xv[pidx(n, i, k)], xjk = xv[pidx(n, j, k)];
                double v1 = xij - xik - xjk, v2 = xik - xij - xjk, v3 = xjk - xij - xik;
                if (v1 > viol) viol = v1;
                if (v2 > viol) viol = v2;
                if (v3 > viol) viol = v3;
            }
        }
    int64_t m = n * (n - 1) / 2;
    for (int64_t p = 0; p < m; ++p) {
        double vu = xv[p] - fv[p] - dflat[p];
        double vl = dflat[p] - xv[p] - fv[p];
        if (vu > viol) viol = vu;
        if (vl > viol) viol = vl;
    }
    return viol;
}
