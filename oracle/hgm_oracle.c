/*
 * hgm_oracle.c -- CPU ORACLE.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
 * --impl reference) may load or execute this library.  The product path
 * (paper_1505_00581_b200/, libhgm.so) never links, imports or calls it, and
 * this file includes nothing from the product.
 *
 * What it is: a plain, slow, fp64 transcription of the paper's matching
 * energy and exact minimisation, in the paper's order and notation:
 *   energy       PAPER.md L117-165  (§2, Eqs. 1-6)
 *   constraints  PAPER.md L174-194  (§2.1, Eqs. 7-8) as read in DESIGN.md R1/R2
 *   recursion    PAPER.md L202-241  (§2.2, Eqs. 9-13)
 *   pruning      PAPER.md L244-249 (§2.2), L312 (§3.2), L376-398 (§3.4, Eq. 14 + minnode)
 * Readings of silent / garbled passages are SURVEY.md §8(c) A1-A16, restated
 * in DESIGN.md §2; each is cited where it is used below.
 *
 * Label convention: scene window nodes are 0..S-1 (sorted by frame, stable);
 * the dummy label epsilon is S (so that "real nodes ascending, then epsilon"
 * is plain integer order, A11).  z[] uses -1 for epsilon at the interface.
 *
 * Parity status: every function here is pinned by tests/test_oracle_*.py
 * (closed forms, worked examples, brute force, invariants).  Nothing is
 * "parity unpinned" except the paper's KTH accuracy, which is out of scope.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    double lambda1, lambda2, lambda3, w_dummy; /* 0.6, 0.2, 5; W^d: A6 */
    int T;                                     /* T = 10 */
} or_params;

typedef struct { /* model chain, one node per occupied frame */
    int M, F;
    const int *t;             /* t(i), frames, strictly increasing */
    const double *x, *y, *f;  /* positions and descriptors f_i [M*F] */
} or_model;

typedef struct { /* scene window nodes sorted by frame */
    int S, F;
    const int *t;
    const double *x, *y, *f;
} or_scene;

static const double OR_PI = 3.14159265358979323846;

/* ---------------------------------------------------------------- Eq. 2 --
 * U(z_i) = ||f_i - f'_{z_i}||  (Euclidean), W^d for the dummy. */
double or_unary(const or_model *m, int i, const or_scene *s, int n, double w_dummy) {
    if (n == s->S) return w_dummy;
    double acc = 0.0;
    for (int k = 0; k < m->F; ++k) {
        double d = m->f[(size_t)i * m->F + k] - s->f[(size_t)n * s->F + k];
        acc += d * d;
    }
    return sqrt(acc);
}

/* ---------------------------------------------------------------- Eq. 5 --
 * Delta(i,j) = |(t(i) - t(j)) - (t'(z_i) - t'(z_j))|. */
double or_delta(double ti, double tj, double tzi, double tzj) {
    return fabs((ti - tj) - (tzi - tzj));
}

/* ---------------------------------------------------------------- Eq. 6 --
 * a(p, v, q): the angle subtended at the MIDDLE point v between v->p and
 * v->q ("angles subtended at point j" for a(i,j,k)), unsigned
 * in [0, pi] (A8), 0 when either ray has zero length (A10). */
double or_angle(double px, double py, double vx, double vy, double qx, double qy) {
    double ux = px - vx, uy = py - vy, wx = qx - vx, wy = qy - vy;
    if ((ux == 0.0 && uy == 0.0) || (wx == 0.0 && wy == 0.0)) return 0.0;
    return atan2(fabs(ux * wy - uy * wx), ux * wx + uy * wy);
}

/* "The difference between angles takes into account the circular domain of
 * angles": wrap to [-pi, pi] (A8). */
double or_wrap(double d) {
    while (d > OR_PI) d -= 2.0 * OR_PI;
    while (d < -OR_PI) d += 2.0 * OR_PI;
    return d;
}

/* D^g(z_i, z_j, z_k) = || (a(i,j,k) - a'(z_i,z_j,z_k), a(j,i,k) - a'(z_j,z_i,z_k)) ||_2
 * for model triple (i, j, k) = (i, i-1, i-2) (Eq. 6). */
double or_dg(const double P[3][2], const double Q[3][2]) {
    /* P = model points (i, j, k); Q = scene points (z_i, z_j, z_k) */
    double e1 = or_wrap(or_angle(P[0][0], P[0][1], P[1][0], P[1][1], P[2][0], P[2][1]) -
                        or_angle(Q[0][0], Q[0][1], Q[1][0], Q[1][1], Q[2][0], Q[2][1]));
    double e2 = or_wrap(or_angle(P[1][0], P[1][1], P[0][0], P[0][1], P[2][0], P[2][1]) -
                        or_angle(Q[1][0], Q[1][1], Q[0][0], Q[0][1], Q[2][0], Q[2][1]));
    return sqrt(e1 * e1 + e2 * e2);
}

/* D(z_i, z_{i-1}, z_{i-2}) = D^t + lambda3 D^g, D^t = Delta(i,i-1) + Delta(i-1,i-2)
 * (Eqs. 3-4).  0 if any label is the dummy (A5).
 * i is the 0-based model index of z_i (i >= 2). */
double or_distortion(const or_model *m, int i, const or_scene *s, int c, int b, int a, double lambda3) {
    if (c == s->S || b == s->S || a == s->S) return 0.0;
    double dt = or_delta(m->t[i], m->t[i - 1], s->t[c], s->t[b]) +
                or_delta(m->t[i - 1], m->t[i - 2], s->t[b], s->t[a]);
    double P[3][2] = {{m->x[i], m->y[i]}, {m->x[i - 1], m->y[i - 1]}, {m->x[i - 2], m->y[i - 2]}};
    double Q[3][2] = {{s->x[c], s->y[c]}, {s->x[b], s->y[b]}, {s->x[a], s->y[a]}};
    return dt + lambda3 * or_dg(P, Q);
}

/* Feasibility of an assignment: SURVEY.md §8(c.1) pair rule + triple rule,
 * i.e. causality (Eq. 7, read as strictly increasing scene frames, A1) and
 * temporal closeness over the hyperedge (Eq. 8 with §3.4's bound, A2), with
 * the dummy forms of A5.  z uses S for epsilon. */
static int real(const or_scene *s, int z) { return z != s->S; }

int or_step_admissible(const or_scene *s, int T, int i, const int *z) {
    /* is z[i] admissible given z[i-1], z[i-2]?  (0-based i) */
    if (i == 0 || !real(s, z[i])) return 1;
    int c = z[i];
    if (i == 1) {
        if (!real(s, z[0])) return 1;
        return s->t[z[0]] < s->t[c] && s->t[c] < s->t[z[0]] + T;
    }
    int b = z[i - 1], a = z[i - 2];
    if (real(s, b) && real(s, a)) return s->t[b] < s->t[c] && s->t[c] < s->t[a] + T;
    if (!real(s, b) && real(s, a)) return s->t[a] < s->t[c] && s->t[c] < s->t[a] + T;
    if (real(s, b) && !real(s, a)) return s->t[b] < s->t[c] && s->t[c] < s->t[b] + T;
    return 1;
}

int or_feasible(const or_model *m, const or_scene *s, const or_params *p, const int *z_in) {
    int *z = (int *)malloc(sizeof(int) * (m->M > 0 ? m->M : 1));
    int ok = 1;
    for (int i = 0; i < m->M; ++i) z[i] = z_in[i] < 0 ? s->S : z_in[i];
    for (int i = 0; i < m->M && ok; ++i) ok = or_step_admissible(s, p->T, i, z);
    free(z);
    return ok;
}

/* E(z) = lambda1 sum_i U(z_i) + lambda2 sum_{i>=3} D(z_i, z_{i-1}, z_{i-2})
 * (Eq. 1 restricted to the chain hyperedges of L200 / Eq. 9,
 * lambdas kept explicit, A7).  z uses -1 for epsilon. */
double or_energy(const or_model *m, const or_scene *s, const or_params *p, const int *z_in) {
    double E = 0.0;
    for (int i = 0; i < m->M; ++i) {
        int c = z_in[i] < 0 ? s->S : z_in[i];
        E += p->lambda1 * or_unary(m, i, s, c, p->w_dummy);
        if (i >= 2) {
            int b = z_in[i - 1] < 0 ? s->S : z_in[i - 1];
            int a = z_in[i - 2] < 0 ? s->S : z_in[i - 2];
            E += p->lambda2 * or_distortion(m, i, s, c, b, a, p->lambda3);
        }
    }
    return E;
}

/* ------------------------------------------------------------ §3.4 ------
 * minnode(f) = inf{n : t'(n) >= f}, S if none (A4 extends
 * it to empty frames and past the end).  Tabulated for frames [t0, t1]. */
typedef struct {
    int t0, t1;
    int *tab;
    int S;
} or_minnode;

static void minnode_build(or_minnode *mn, const or_scene *s, int T) {
    mn->S = s->S;
    mn->t0 = s->S ? s->t[0] : 0;
    mn->t1 = (s->S ? s->t[s->S - 1] : 0) + T + 2;
    int nf = mn->t1 - mn->t0 + 1;
    mn->tab = (int *)malloc(sizeof(int) * nf);
    for (int f = mn->t0; f <= mn->t1; ++f) {
        int n = 0;
        while (n < s->S && s->t[n] < f) ++n; /* the definition, written out */
        mn->tab[f - mn->t0] = n;
    }
}
static int minnode(const or_minnode *mn, int f) {
    if (f <= mn->t0) return 0;
    if (f > mn->t1) return mn->S;
    return mn->tab[f - mn->t0];
}

/* exported for the minnode pins (Fig. 6 caption) */
int or_minnode_at(const or_scene *s, int T, int f) {
    or_minnode mn;
    minnode_build(&mn, s, T);
    int r = minnode(&mn, f);
    free(mn.tab);
    return r;
}

/* --------------------------------------------------------- Eqs. 10-13 --
 * The exact DP.  alpha_i(z_{i-1}, z_{i-2}) is held densely as an (S+1)x(S+1)
 * table (PAPER.md: "a series of 2D tables of size SxS", plus the
 * dummy row/column); beta_i is kept only for the admissible cross-section
 * ("a cross section of size ~SxT").
 *
 * Admissible states (z_{i-1}, z_{i-2}) = (b, a): b real and a real with
 * t'(a) < t'(b) < t'(a) + T ("z_{i-2} is restricted to the interval
 * ]z_{i-1}-T, z_{i-1}[", in frames, A1/A2); or either is the
 * dummy (A5).
 *
 * Candidates z_i = c for state (b, a) (PAPER.md L393-398 with A1, A3, A5):
 *   lo = minnode(t'(b) + 1)   (or t'(a)+1 if b = eps; 0 if both eps)
 *   hi = minnode(t'(a) + T)   (or t'(b)+T if a = eps; S if both eps)
 *   c = lo .. hi-1 ascending, then eps; the first strict minimum wins (A11).
 */
typedef struct {
    int *off; /* per b in 0..S: start in val[] */
    int *lo;  /* per b: first real a of its admissible range */
    int *n;   /* per b: number of real a (eps is slot n[b]) */
    int *val;
} or_beta;

static int states_lo(const or_minnode *mn, const or_scene *s, int T, int b) {
    return b == s->S ? 0 : minnode(mn, s->t[b] - T + 1);
}
static int states_hi(const or_minnode *mn, const or_scene *s, int b) {
    return b == s->S ? s->S : minnode(mn, s->t[b]);
}

int or_match(const or_model *m, const or_scene *s, const or_params *p, double *E_dp, double *E_re,
             double *A, int *z_out) {
    const int M = m->M, S = s->S, S1 = S + 1, T = p->T, EPS = S;
    if (M < 1) return 1;
    or_minnode mn;
    minnode_build(&mn, s, T);

    /* §3.3: unary look-up table U[i][n], n = S is the dummy */
    double *U = (double *)malloc(sizeof(double) * (size_t)M * S1);
    for (int i = 0; i < M; ++i)
        for (int n = 0; n <= S; ++n) U[(size_t)i * S1 + n] = or_unary(m, i, s, n, p->w_dummy);

    double *a_next = (double *)malloc(sizeof(double) * (size_t)S1 * S1); /* alpha_{i+1} */
    double *a_cur = (double *)malloc(sizeof(double) * (size_t)S1 * S1);  /* alpha_i */
    for (size_t k = 0; k < (size_t)S1 * S1; ++k) a_next[k] = 0.0; /* alpha_{M+1} := 0 (Eq. 11) */

    /* beta storage, one table per step i = 3..M (1-based), cross-section only */
    int nsteps = M >= 3 ? M - 2 : 0;
    or_beta *beta = (or_beta *)calloc(nsteps > 0 ? nsteps : 1, sizeof(or_beta));
    for (int st = 0; st < nsteps; ++st) {
        beta[st].off = (int *)malloc(sizeof(int) * S1);
        beta[st].lo = (int *)malloc(sizeof(int) * S1);
        beta[st].n = (int *)malloc(sizeof(int) * S1);
        int tot = 0;
        for (int b = 0; b <= S; ++b) {
            beta[st].lo[b] = states_lo(&mn, s, T, b);
            beta[st].n[b] = states_hi(&mn, s, b) - beta[st].lo[b];
            if (beta[st].n[b] < 0) beta[st].n[b] = 0;
            beta[st].off[b] = tot;
            tot += beta[st].n[b] + 1;
        }
        beta[st].val = (int *)malloc(sizeof(int) * (size_t)(tot > 0 ? tot : 1));
    }

    /* model angles at the chain triangles are constants of each step i */
    for (int i = M - 1; i >= 2; --i) { /* 0-based i: paper's i = i+1, from M down to 3 */
        or_beta *bt = &beta[i - 2];
        for (size_t k = 0; k < (size_t)S1 * S1; ++k) a_cur[k] = INFINITY; /* inadmissible */
        for (int b = 0; b <= S; ++b) {
            for (int ai = 0; ai <= bt->n[b]; ++ai) {
                int a = ai < bt->n[b] ? bt->lo[b] + ai : EPS;
                /* candidate loop bounds (A1/A5) */
                int lo, hi;
                if (b != EPS) lo = minnode(&mn, s->t[b] + 1);
                else if (a != EPS) lo = minnode(&mn, s->t[a] + 1);
                else lo = 0;
                if (a != EPS) hi = minnode(&mn, s->t[a] + T);
                else if (b != EPS) hi = minnode(&mn, s->t[b] + T);
                else hi = S;
                double best = INFINITY;
                int arg = -2;
                for (int c = lo; c <= hi; ++c) {
                    int cc = c < hi ? c : EPS; /* reals ascending, then eps (A11) */
                    /* Eq. 10: U(z_i) + D(z_i, z_{i-1}, z_{i-2}) + alpha_{i+1}(z_i, z_{i-1}) */
                    double v = p->lambda1 * U[(size_t)i * S1 + cc] +
                               p->lambda2 * or_distortion(m, i, s, cc, b, a, p->lambda3) +
                               a_next[(size_t)cc * S1 + b];
                    if (v < best) { best = v; arg = cc; }
                }
                a_cur[(size_t)b * S1 + a] = best;
                bt->val[bt->off[b] + ai] = arg;
            }
        }
        double *tmp = a_next; a_next = a_cur; a_cur = tmp; /* a_next := alpha_i */
    }
    /* a_next now holds alpha_3 (or 0 when M <= 2: alpha_3 := 0, A9) */

    int *z = (int *)malloc(sizeof(int) * M);
    double best = INFINITY;
    if (M == 1) { /* A9: min over z_1 of lambda1 U(z_1) */
        for (int c = 0; c <= S; ++c) {
            double v = p->lambda1 * U[c];
            if (v < best) { best = v; z[0] = c; }
        }
    } else {
        /* Eq. 13: (z1, z2) = argmin U(z1) + U(z2) + alpha_3(z2, z1), lexicographic (A11),
         * over pairs obeying the pair rule (Eq. 7/8 for the first hyperedge, A1/A2). */
        for (int z1 = 0; z1 <= S; ++z1) {
            for (int z2 = 0; z2 <= S; ++z2) {
                if (z1 != EPS && z2 != EPS && !(s->t[z1] < s->t[z2] && s->t[z2] < s->t[z1] + T)) continue;
                double v = p->lambda1 * U[z1] + p->lambda1 * U[(size_t)S1 + z2] + a_next[(size_t)z2 * S1 + z1];
                if (v < best) { best = v; z[0] = z1; z[1] = z2; }
            }
        }
        /* Eq. 12: backtracking z_i = beta_i(z_{i-1}, z_{i-2}) */
        for (int i = 2; i < M; ++i) {
            or_beta *bt = &beta[i - 2];
            int b = z[i - 1], a = z[i - 2];
            int ai = (a == EPS) ? bt->n[b] : a - bt->lo[b];
            z[i] = bt->val[bt->off[b] + ai];
        }
    }
    for (int i = 0; i < M; ++i) z_out[i] = z[i] == EPS ? -1 : z[i];
    *E_dp = best;
    *E_re = or_energy(m, s, p, z_out);
    double acc = 0.0; /* appearance distance: sum of U only, unweighted (A14) */
    for (int i = 0; i < M; ++i) acc += U[(size_t)i * S1 + z[i]];
    *A = acc;

    for (int st = 0; st < nsteps; ++st) {
        free(beta[st].off); free(beta[st].lo); free(beta[st].n); free(beta[st].val);
    }
    free(beta); free(z); free(a_next); free(a_cur); free(U); free(mn.tab);
    return 0;
}

/* ------------------------------------------------------------ batches ---
 * Independent (model, window) jobs over one sorted scene, on a thread pool
 * (one job per task, SURVEY.md §8(d) "Oracle timing"). */
typedef struct {
    const or_model *models;
    const or_scene *scene;
    const or_params *p;
    const int *job_model, *job_wb, *job_we;
    double *E_dp, *E_re, *A;
    int *z;
    int Mmax, n_jobs;
    int next;
    pthread_mutex_t mu;
} or_pool;

static void *or_worker(void *arg) {
    or_pool *P = (or_pool *)arg;
    for (;;) {
        pthread_mutex_lock(&P->mu);
        int j = P->next++;
        pthread_mutex_unlock(&P->mu);
        if (j >= P->n_jobs) break;
        const or_model *m = &P->models[P->job_model[j]];
        int wb = P->job_wb[j], we = P->job_we[j];
        or_scene w = {we - wb, P->scene->F, P->scene->t + wb, P->scene->x + wb, P->scene->y + wb,
                      P->scene->f + (size_t)wb * P->scene->F};
        int *zz = P->z + (size_t)j * P->Mmax;
        for (int i = 0; i < P->Mmax; ++i) zz[i] = -1;
        or_match(m, &w, P->p, &P->E_dp[j], &P->E_re[j], &P->A[j], zz);
        for (int i = 0; i < m->M; ++i)
            if (zz[i] >= 0) zz[i] += wb; /* report scene-sorted node index */
    }
    return NULL;
}

int or_match_batch(const or_model *models, const or_scene *scene, const or_params *p, int n_jobs,
                   const int *job_model, const int *job_wb, const int *job_we, int n_threads,
                   double *E_dp, double *E_re, double *A, int *z, int Mmax) {
    or_pool P = {models, scene, p, job_model, job_wb, job_we, E_dp, E_re, A, z, Mmax, n_jobs, 0};
    pthread_mutex_init(&P.mu, NULL);
    if (n_threads < 1) n_threads = 1;
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * n_threads);
    for (int k = 0; k < n_threads; ++k) pthread_create(&th[k], NULL, or_worker, &P);
    for (int k = 0; k < n_threads; ++k) pthread_join(th[k], NULL);
    free(th);
    pthread_mutex_destroy(&P.mu);
    return 0;
}
