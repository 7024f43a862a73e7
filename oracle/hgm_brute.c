/*
 * hgm_brute.c -- BRUTE-FORCE ENUMERATOR.  TEST INFRASTRUCTURE ONLY.
 *
 * Pins the oracle DP (hgm_oracle.c) on tiny instances.  It shares nothing
 * with the DP's loop bounds: it walks the feasible set Z of SURVEY.md
 * §8(c.1) depth-first, testing the DECLARATIVE per-position predicate
 * (or_step_admissible: pair rule + triple rule, written from the text of
 * Eqs. 7-8 under readings A1/A2/A5), and accumulates the energy of Eq. 1
 * term by term.  The predicate is prefix-closed, so DFS over
 * admissible extensions enumerates Z exactly.  Labels are tried in the order
 * 0 < 1 < ... < S-1 < eps and the FIRST strict minimum is kept, so the result
 * is the lexicographically smallest minimiser (A11).
 *
 * Branch and bound: every term is >= 0 (U >= 0, W^d >= 0, D >= 0), so a
 * prefix whose partial energy is already >= the best leaf cannot produce a
 * strictly smaller leaf and is skipped.  This changes nothing in the result.
 */
#include <math.h>
#include <stdlib.h>

typedef struct { double lambda1, lambda2, lambda3, w_dummy; int T; } or_params;
typedef struct { int M, F; const int *t; const double *x, *y, *f; } or_model;
typedef struct { int S, F; const int *t; const double *x, *y, *f; } or_scene;

double or_unary(const or_model *m, int i, const or_scene *s, int n, double w_dummy);
double or_distortion(const or_model *m, int i, const or_scene *s, int c, int b, int a, double lambda3);
int or_step_admissible(const or_scene *s, int T, int i, const int *z);

typedef struct {
    const or_model *m;
    const or_scene *s;
    const or_params *p;
    const double *U; /* U[i][n], n = S is eps -- a cache of Eq. 2, nothing else */
    int *z, *zbest;
    double best;
    long long leaves;
    int prune;
} br_ctx;

static void dfs(br_ctx *C, int i, double E) {
    const int M = C->m->M, S = C->s->S;
    if (i == M) {
        ++C->leaves;
        if (E < C->best) {
            C->best = E;
            for (int k = 0; k < M; ++k) C->zbest[k] = C->z[k];
        }
        return;
    }
    for (int c = 0; c <= S; ++c) {
        C->z[i] = c;
        if (!or_step_admissible(C->s, C->p->T, i, C->z)) continue;
        double e = C->p->lambda1 * C->U[(size_t)i * (S + 1) + c];
        if (i >= 2) e += C->p->lambda2 * or_distortion(C->m, i, C->s, c, C->z[i - 1], C->z[i - 2], C->p->lambda3);
        if (C->prune && E + e >= C->best) continue;
        dfs(C, i + 1, E + e);
    }
}

int or_brute(const or_model *m, const or_scene *s, const or_params *p, int prune, double *E, int *z_out,
             long long *n_leaves) {
    const int M = m->M, S = s->S;
    double *U = (double *)malloc(sizeof(double) * (size_t)M * (S + 1));
    for (int i = 0; i < M; ++i)
        for (int n = 0; n <= S; ++n) U[(size_t)i * (S + 1) + n] = or_unary(m, i, s, n, p->w_dummy);
    int *z = (int *)malloc(sizeof(int) * M), *zb = (int *)malloc(sizeof(int) * M);
    for (int k = 0; k < M; ++k) zb[k] = S;
    br_ctx C = {m, s, p, U, z, zb, INFINITY, 0, prune};
    dfs(&C, 0, 0.0);
    for (int k = 0; k < M; ++k) z_out[k] = zb[k] == S ? -1 : zb[k];
    *E = C.best;
    *n_leaves = C.leaves;
    free(U); free(z); free(zb);
    return 0;
}
