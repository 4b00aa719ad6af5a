/*
 * nbx_oracle.c -- CPU restatement of the NBNXM hot path.  TEST INFRASTRUCTURE ONLY
 * (see nbx_oracle.h for who may use it).  Plain C99 + OpenMP, compiled with
 * -ffp-contract=off so every fused multiply-add below is an explicit fmaf().
 *
 * Reference anchors (the reference only prices these steps, it never computes them):
 *   grid + pair search  KernelKind.PAIR_SEARCH   costs.py:32,163   pipeline.py:226-230
 *   dynamic prune       KernelKind.PRUNE_ONLY    costs.py:31,162   pipeline.py:223-235
 *   force kernel        KernelKind.NBNXM_LOCAL/NONLOCAL costs.py:29-30  pipeline.py:231,384
 *   F buffer op         KernelKind.REDUCE_FORCES costs.py:41,172   pipeline.py:250-254
 * The arithmetic follows DESIGN.md sections "Physics", "Grid", "Search", "Prune", "Force".
 */
#include "nbx_oracle.h"

#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define FILLER_COORD (-1.0e5f)
#define BB_EMPTY 1.0e30f
#define R2MIN 1.0e-6f

/* ------------------------------------------------------------------ constants */

static double ewald_beta(double rc, double rtol)
{
    /* smallest beta with erfc(beta rc) <= rtol: doubling bracket then 60 bisections */
    double lo = 0.0, hi = 5.0;
    while (erfc(hi * rc) > rtol) hi *= 2.0;
    for (int it = 0; it < 60; it++) {
        double mid = 0.5 * (lo + hi);
        if (erfc(mid * rc) > rtol) lo = mid; else hi = mid;
    }
    return 0.5 * (lo + hi);
}

int ora_derive_consts(const nbx_params* p, nbx_consts* c)
{
    double rc = p->rc;
    memset(c, 0, sizeof(*c));
    c->epsfac = (float)(138.935458 / (double)p->epsilon_r);
    double krf;
    if (p->epsilon_rf == 0.0f)
        krf = 1.0 / (2.0 * rc * rc * rc);
    else
        krf = ((double)p->epsilon_rf - (double)p->epsilon_r)
              / ((2.0 * (double)p->epsilon_rf + (double)p->epsilon_r) * rc * rc * rc);
    c->k_rf = (float)krf;
    c->c_rf = (float)(1.0 / rc + krf * rc * rc);
    const int ew = p->coulomb_type == NBX_COULOMB_EWALD || p->coulomb_type == NBX_COULOMB_EWALD_TAB;
    double beta = ew ? ewald_beta(rc, p->ewald_rtol) : 0.0;
    c->beta = (float)beta;
    c->sh_ewald = ew ? (float)(erfc(beta * rc) / rc) : 0.0f;
    if (p->coulomb_type == NBX_COULOMB_EWALD_TAB) {
        c->tab_scale = (float)(400.0 * beta > 600.0 ? 400.0 * beta : 600.0);
        c->tab_n = (int32_t)ceil(rc * (double)c->tab_scale) + 2;
    }
    c->sh_lj6 = (float)(1.0 / (rc * rc * rc * rc * rc * rc));
    c->sh_lj12 = (float)(1.0 / (rc * rc * rc * rc * rc * rc * rc * rc * rc * rc * rc * rc));
    c->rc2 = (float)(rc * rc);
    c->rlo2 = (float)((double)p->rlist_outer * (double)p->rlist_outer);
    c->rli2 = (float)((double)p->rlist_inner * (double)p->rlist_inner);
    if (p->lj_modifier == NBX_LJ_FORCE_SWITCH) {
        const double r1 = p->rvdw_switch, d = rc - r1;
        double A[2], B[2], C[2];
        const double al[2] = {6.0, 12.0};
        for (int k = 0; k < 2; k++) {
            const double a = al[k], rca2 = pow(rc, a + 2.0);
            A[k] = -a * ((a + 4.0) * rc - (a + 1.0) * r1) / (rca2 * d * d);
            B[k] = a * ((a + 3.0) * rc - (a + 1.0) * r1) / (rca2 * d * d * d);
            C[k] = pow(rc, -a) - A[k] / 3.0 * d * d * d - B[k] / 4.0 * d * d * d * d;
        }
        c->fsw_r1 = (float)r1;
        c->fsw_a6 = (float)(A[0] / 6.0);
        c->fsw_b6 = (float)(B[0] / 6.0);
        c->fsw_a12 = (float)(A[1] / 12.0);
        c->fsw_b12 = (float)(B[1] / 12.0);
        c->fsw_p6 = (float)(A[0] / 3.0);
        c->fsw_q6 = (float)(B[0] / 4.0);
        c->fsw_p12 = (float)(A[1] / 3.0);
        c->fsw_q12 = (float)(B[1] / 4.0);
        c->fsw_c6 = (float)C[0];
        c->fsw_c12 = (float)C[1];
    }
    if (!(p->rc > 0.0f) || p->rlist_inner < p->rc || p->rlist_outer < p->rlist_inner) return 1;
    if (p->lj_modifier == NBX_LJ_FORCE_SWITCH && !(p->rvdw_switch >= 0.0f && p->rvdw_switch < p->rc)) return 1;
    return 0;
}

/* beta^3 G(beta^2 r^2) = (erf(beta r)/r - 2 beta/sqrt(pi) exp(-beta^2 r^2)) / r^2, with its
 * series (2 beta^3/sqrt(pi)) (2/3 - 2z/5 + z^2/7 - z^3/27 + z^4/132) below z = 1e-2 */
static double ewald_fcorr(double beta, double r)
{
    const double z = beta * beta * r * r, b3 = beta * beta * beta, tsp = 2.0 / sqrt(M_PI);
    if (z < 1e-2) return tsp * b3 * (2.0 / 3.0 + z * (-2.0 / 5.0 + z * (1.0 / 7.0 + z * (-1.0 / 27.0 + z / 132.0))));
    return (erf(beta * r) / r - tsp * beta * exp(-z)) / (r * r);
}

static double ewald_vcorr(double beta, double r)
{
    if (r == 0.0) return 2.0 * beta / sqrt(M_PI);
    return erf(beta * r) / r;
}

int ora_ewald_table(const nbx_consts* c, float* ftab, float* vtab)
{
    const int n = c->tab_n;
    if (n < 2 || !(c->tab_scale > 0.0f)) return 1;
    const double beta = c->beta, h = 1.0 / (double)c->tab_scale;
    for (int k = 0; k < n; k++) {
        ftab[2 * k] = (float)ewald_fcorr(beta, k * h);
        vtab[2 * k] = (float)ewald_vcorr(beta, k * h);
    }
    for (int k = 0; k < n; k++) {
        ftab[2 * k + 1] = (k + 1 < n) ? ftab[2 * k + 2] - ftab[2 * k] : 0.0f;
        vtab[2 * k + 1] = (k + 1 < n) ? vtab[2 * k + 2] - vtab[2 * k] : 0.0f;
    }
    return 0;
}

/* linear interpolation of a (value, difference) table at r = r2 * rinv, identical op
 * sequence to tab_lookup() in paper_2405_01420_b200/csrc/pairmath.cuh: the floor comes from
 * adding 2^23 - 1/2 (exact for rs >= 1/2, which R2MIN and tab_scale >= 600 guarantee) */
static inline float tab_interp(const float* tab, float r2, float rinv, const nbx_consts* c)
{
    const float r2c = fminf(r2, c->rc2);
    const float rs = r2c * (rinv * c->tab_scale);
    const float t = rs + 8388607.5f;
    uint32_t tb;
    memcpy(&tb, &t, 4);
    const int idx = (int)(tb - 0x4B000000u);
    const float fr = rs - (t - 8388608.0f);
    return fmaf(fr, tab[2 * idx + 1], tab[2 * idx]);
}

double ora_self_energy(const nbx_params* p, double sumq2)
{
    nbx_consts c;
    ora_derive_consts(p, &c);
    if (p->coulomb_type == NBX_COULOMB_EWALD || p->coulomb_type == NBX_COULOMB_EWALD_TAB)
        return -(double)c.epsfac * sumq2 * (double)c.beta / sqrt(M_PI);
    return -0.5 * (double)c.epsfac * (double)c.c_rf * sumq2;
}

/* Ewald real-space rational approximations, fitted by tools/fit_ewald.py:
 *   G(z) ~ erf(sqrt z)/z^1.5 - 2/sqrt(pi) exp(-z)/z   (max rel err 5.0e-7 on [0,12.5])
 *   H(z) ~ erf(sqrt z)/sqrt z                          (max rel err 5.3e-7 on [0,12.5]) */
static const float EW_GP[6] = {0.752252758f, -0.0231583007f, 0.0169008784f, 9.68796448e-05f,
                               3.47007081e-05f, -3.8098932e-07f};
static const float EW_GQ[6] = {1.0f, 0.569215298f, 0.149706319f, 0.0235451832f, 0.00233585062f,
                               0.000141900193f};
static const float EW_HP[7] = {1.12837923f, 0.182699338f, 0.0532767773f, 0.00366060762f, 0.000346426154f, 3.80142114e-06f, -8.10354006e-09f};
static const float EW_HQ[6] = {1.0f, 0.49524644f, 0.112297274f, 0.0149619607f, 0.00122577278f, 5.49911565e-05f};

float ora_ewald_G(float z)
{
    float n = EW_GP[5], d = EW_GQ[5];
    for (int k = 4; k >= 0; k--) { n = fmaf(n, z, EW_GP[k]); d = fmaf(d, z, EW_GQ[k]); }
    return n / d;
}

float ora_ewald_H(float z)
{
    float n = EW_HP[6], d = EW_HQ[5];
    for (int k = 5; k >= 0; k--) n = fmaf(n, z, EW_HP[k]);
    for (int k = 4; k >= 0; k--) d = fmaf(d, z, EW_HQ[k]);
    return n / d;
}

/* ------------------------------------------------------------------ grid */

struct ora_grid {
    int n, ncx, ncy, ncol, nslots, nsci;
    float box[3], lo[3], size[3], inv_cell[2];
    int pbc[3];
    int* col_start; /* [ncol+1] */
    int* order;     /* [nslots] input index or -1 */
    int* gid;       /* [nslots] */
    float* xq;      /* [nslots*4] */
    int* type;      /* [nslots] */
    float* wrapk;   /* [nslots*3] */
    float* bb_ci;   /* [nci*6] lo xyz, hi xyz */
    float* bb_cj;   /* [ncj*6] */
    float* bb_sci;  /* [nsci*6] */
    int* nreal_ci;
    int* nreal_cj;
    int* nreal_sci;
    int* exlo_ci; /* partner gid range per i-cluster */
    int* exhi_ci;
    int* glo_cj; /* gid range per j-cluster */
    int* ghi_cj;
    const int* excl_offsets; /* borrowed, global */
    const int* excl_gids;
    double sumq2;
};

static inline uint32_t ordkey(float f)
{
    uint32_t u;
    memcpy(&u, &f, 4);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

void ora_grid_dims(const float size[3], double density, int* ncx, int* ncy, float inv_cell[2])
{
    double s = cbrt(32.0 / density);
    int nx = (int)floor((double)size[0] / s + 0.5);
    int ny = (int)floor((double)size[1] / s + 0.5);
    if (nx < 1) nx = 1;
    if (ny < 1) ny = 1;
    *ncx = nx;
    *ncy = ny;
    inv_cell[0] = (float)((double)nx / (double)size[0]);
    inv_cell[1] = (float)((double)ny / (double)size[1]);
}

static inline int cell_index(float xw, float lo, float inv, int nc)
{
    float t = floorf((xw - lo) * inv);
    if (!(t >= 0.0f)) return 0; /* also catches NaN */
    if (t > (float)(nc - 1)) return nc - 1;
    return (int)t;
}

typedef struct { uint64_t key; int idx; } sortrec;

static int cmp_sortrec(const void* a, const void* b)
{
    const sortrec* x = (const sortrec*)a;
    const sortrec* y = (const sortrec*)b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    return x->idx - y->idx;
}

typedef struct { uint32_t key; int idx; } sortrec32;

static int cmp_sortrec32(const void* a, const void* b)
{
    const sortrec32* x = (const sortrec32*)a;
    const sortrec32* y = (const sortrec32*)b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    return x->idx - y->idx;
}

/* sort `cnt` atom input indices by (key of coordinate dim, input index) */
static void sort_by_dim(int* idx, int cnt, const float* xw, int dim)
{
    sortrec32 r[32];
    for (int k = 0; k < cnt; k++) { r[k].key = ordkey(xw[3 * idx[k] + dim]); r[k].idx = idx[k]; }
    qsort(r, cnt, sizeof(sortrec32), cmp_sortrec32);
    for (int k = 0; k < cnt; k++) idx[k] = r[k].idx;
}

static void bb_init(float* b) { b[0] = b[1] = b[2] = BB_EMPTY; b[3] = b[4] = b[5] = -BB_EMPTY; }

static void bb_union(float* b, const float* o)
{
    for (int d = 0; d < 3; d++) {
        b[d] = fminf(b[d], o[d]);
        b[3 + d] = fmaxf(b[3 + d], o[3 + d]);
    }
}

ora_grid* ora_grid_build(int n, const float* x, const int* gid_in, const float* q_global,
                         const int* type_global, const int* excl_offsets, const int* excl_gids,
                         const float box[3], const int pbc[3], const float lo[3],
                         const float size[3], double density)
{
    ora_grid* g = (ora_grid*)calloc(1, sizeof(ora_grid));
    g->n = n;
    for (int d = 0; d < 3; d++) {
        g->box[d] = box[d]; g->lo[d] = lo[d]; g->size[d] = size[d]; g->pbc[d] = pbc[d];
    }
    g->excl_offsets = excl_offsets;
    g->excl_gids = excl_gids;
    ora_grid_dims(size, density, &g->ncx, &g->ncy, g->inv_cell);
    g->ncol = g->ncx * g->ncy;

    float invL[3];
    for (int d = 0; d < 3; d++) invL[d] = (float)(1.0 / (double)box[d]);
    float* xw = (float*)malloc(sizeof(float) * 3 * (size_t)(n > 0 ? n : 1));
    float* kk = (float*)malloc(sizeof(float) * 3 * (size_t)(n > 0 ? n : 1));
    sortrec* rec = (sortrec*)malloc(sizeof(sortrec) * (size_t)(n > 0 ? n : 1));
    int* colcnt = (int*)calloc((size_t)g->ncol, sizeof(int));
    for (int a = 0; a < n; a++) {
        for (int d = 0; d < 3; d++) {
            float xv = x[3 * a + d];
            float k = pbc[d] ? floorf(xv * invL[d]) : 0.0f;
            kk[3 * a + d] = k;
            xw[3 * a + d] = fmaf(-k, box[d], xv);
        }
        int cx = cell_index(xw[3 * a + 0], lo[0], g->inv_cell[0], g->ncx);
        int cy = cell_index(xw[3 * a + 1], lo[1], g->inv_cell[1], g->ncy);
        int col = cx * g->ncy + cy;
        colcnt[col]++;
        rec[a].key = ((uint64_t)(uint32_t)col << 32) | ordkey(xw[3 * a + 2]);
        rec[a].idx = a;
    }
    qsort(rec, (size_t)n, sizeof(sortrec), cmp_sortrec);

    g->col_start = (int*)malloc(sizeof(int) * (size_t)(g->ncol + 1));
    g->col_start[0] = 0;
    for (int c = 0; c < g->ncol; c++) g->col_start[c + 1] = g->col_start[c] + ((colcnt[c] + 31) / 32) * 32;
    g->nslots = g->col_start[g->ncol];
    g->nsci = g->nslots / 32;
    int ns = g->nslots, nci = ns / 4, ncj = ns / 8, nsci = g->nsci;
    g->order = (int*)malloc(sizeof(int) * (size_t)(ns + 1));
    g->gid = (int*)malloc(sizeof(int) * (size_t)(ns + 1));
    g->xq = (float*)malloc(sizeof(float) * 4 * (size_t)(ns + 1));
    g->type = (int*)malloc(sizeof(int) * (size_t)(ns + 1));
    g->wrapk = (float*)malloc(sizeof(float) * 3 * (size_t)(ns + 1));
    for (int s = 0; s < ns; s++) g->order[s] = -1;

    /* slab sub-sort: y halves of 16 -> x quarters of 8 (j-clusters) -> z halves of 4 */
    int pos = 0; /* position in sorted rec */
    for (int c = 0; c < g->ncol; c++) {
        int cnt = colcnt[c];
        for (int s0 = 0; s0 < cnt; s0 += 32) {
            int m = cnt - s0 < 32 ? cnt - s0 : 32;
            int members[32];
            for (int k = 0; k < m; k++) members[k] = rec[pos + s0 + k].idx;
            int slab_slot = g->col_start[c] + s0;
            sort_by_dim(members, m, xw, 1);
            for (int h = 0; h < 2; h++) {
                int hb = h * 16, hc = h == 0 ? (m < 16 ? m : 16) : (m > 16 ? m - 16 : 0);
                int* hm = members + hb;
                sort_by_dim(hm, hc, xw, 0);
                for (int qd = 0; qd < 2; qd++) {
                    int qb = qd * 8, qc = qd == 0 ? (hc < 8 ? hc : 8) : (hc > 8 ? hc - 8 : 0);
                    int* qm = hm + qb;
                    sort_by_dim(qm, qc, xw, 2);
                    for (int ic = 0; ic < 2; ic++) {
                        int ib = ic * 4, icnt = ic == 0 ? (qc < 4 ? qc : 4) : (qc > 4 ? qc - 4 : 0);
                        for (int k = 0; k < icnt; k++)
                            g->order[slab_slot + hb + qb + ib + k] = qm[ib + k];
                    }
                }
            }
        }
        pos += cnt;
    }
    g->sumq2 = 0.0;
    for (int s = 0; s < ns; s++) {
        int a = g->order[s];
        if (a >= 0) {
            int gg = gid_in ? gid_in[a] : a;
            g->gid[s] = gg;
            for (int d = 0; d < 3; d++) { g->xq[4 * s + d] = xw[3 * a + d]; g->wrapk[3 * s + d] = kk[3 * a + d]; }
            g->xq[4 * s + 3] = q_global[gg];
            g->type[s] = type_global[gg];
            g->sumq2 += (double)q_global[gg] * (double)q_global[gg];
        } else {
            g->gid[s] = -1;
            for (int d = 0; d < 3; d++) { g->xq[4 * s + d] = FILLER_COORD; g->wrapk[3 * s + d] = 0.0f; }
            g->xq[4 * s + 3] = 0.0f;
            g->type[s] = 0;
        }
    }
    /* bounding boxes, real counts, exclusion / gid ranges */
    g->bb_ci = (float*)malloc(sizeof(float) * 6 * (size_t)(nci + 1));
    g->bb_cj = (float*)malloc(sizeof(float) * 6 * (size_t)(ncj + 1));
    g->bb_sci = (float*)malloc(sizeof(float) * 6 * (size_t)(nsci + 1));
    g->nreal_ci = (int*)calloc((size_t)nci + 1, sizeof(int));
    g->nreal_cj = (int*)calloc((size_t)ncj + 1, sizeof(int));
    g->nreal_sci = (int*)calloc((size_t)nsci + 1, sizeof(int));
    g->exlo_ci = (int*)malloc(sizeof(int) * (size_t)(nci + 1));
    g->exhi_ci = (int*)malloc(sizeof(int) * (size_t)(nci + 1));
    g->glo_cj = (int*)malloc(sizeof(int) * (size_t)(ncj + 1));
    g->ghi_cj = (int*)malloc(sizeof(int) * (size_t)(ncj + 1));
    for (int ci = 0; ci < nci; ci++) {
        float* b = g->bb_ci + 6 * ci;
        bb_init(b);
        int elo = 0x7fffffff, ehi = -1;
        for (int i = 0; i < 4; i++) {
            int s = 4 * ci + i;
            if (g->order[s] < 0) continue;
            g->nreal_ci[ci]++;
            for (int d = 0; d < 3; d++) {
                b[d] = fminf(b[d], g->xq[4 * s + d]);
                b[3 + d] = fmaxf(b[3 + d], g->xq[4 * s + d]);
            }
            int gg = g->gid[s];
            for (int e = excl_offsets[gg]; e < excl_offsets[gg + 1]; e++) {
                int p = excl_gids[e];
                if (p < elo) elo = p;
                if (p > ehi) ehi = p;
            }
        }
        g->exlo_ci[ci] = elo;
        g->exhi_ci[ci] = ehi;
    }
    for (int cj = 0; cj < ncj; cj++) {
        float* b = g->bb_cj + 6 * cj;
        bb_init(b);
        bb_union(b, g->bb_ci + 6 * (2 * cj));
        bb_union(b, g->bb_ci + 6 * (2 * cj + 1));
        g->nreal_cj[cj] = g->nreal_ci[2 * cj] + g->nreal_ci[2 * cj + 1];
        int glo = 0x7fffffff, ghi = -1;
        for (int j = 0; j < 8; j++) {
            int gg = g->gid[8 * cj + j];
            if (gg < 0) continue;
            if (gg < glo) glo = gg;
            if (gg > ghi) ghi = gg;
        }
        g->glo_cj[cj] = glo;
        g->ghi_cj[cj] = ghi;
    }
    for (int sc = 0; sc < nsci; sc++) {
        float* b = g->bb_sci + 6 * sc;
        bb_init(b);
        for (int k = 0; k < 8; k++) {
            bb_union(b, g->bb_ci + 6 * (8 * sc + k));
            g->nreal_sci[sc] += g->nreal_ci[8 * sc + k];
        }
    }
    free(xw); free(kk); free(rec); free(colcnt);
    return g;
}

void ora_grid_free(ora_grid* g)
{
    if (!g) return;
    free(g->col_start); free(g->order); free(g->gid); free(g->xq); free(g->type); free(g->wrapk);
    free(g->bb_ci); free(g->bb_cj); free(g->bb_sci); free(g->nreal_ci); free(g->nreal_cj);
    free(g->nreal_sci); free(g->exlo_ci); free(g->exhi_ci); free(g->glo_cj); free(g->ghi_cj);
    free(g);
}

int ora_grid_nslots(const ora_grid* g) { return g->nslots; }
int ora_grid_ncx(const ora_grid* g) { return g->ncx; }
int ora_grid_ncy(const ora_grid* g) { return g->ncy; }
double ora_grid_sumq2(const ora_grid* g) { return g->sumq2; }

void ora_grid_export(const ora_grid* g, int* order, float* xq, int* type, int* gid)
{
    size_t ns = (size_t)g->nslots;
    if (order) memcpy(order, g->order, ns * sizeof(int));
    if (xq) memcpy(xq, g->xq, ns * 4 * sizeof(float));
    if (type) memcpy(type, g->type, ns * sizeof(int));
    if (gid) memcpy(gid, g->gid, ns * sizeof(int));
}

void ora_grid_put_x(ora_grid* g, const float* x)
{
    for (int s = 0; s < g->nslots; s++) {
        int a = g->order[s];
        if (a < 0) continue;
        for (int d = 0; d < 3; d++) g->xq[4 * s + d] = fmaf(-g->wrapk[3 * s + d], g->box[d], x[3 * a + d]);
    }
}

void ora_grid_get_f(const ora_grid* g, const double* f_slots, float* f_out, int accumulate)
{
    for (int s = 0; s < g->nslots; s++) {
        int a = g->order[s];
        if (a < 0) continue;
        for (int d = 0; d < 3; d++) {
            float v = (float)f_slots[3 * s + d];
            f_out[3 * a + d] = accumulate ? f_out[3 * a + d] + v : v;
        }
    }
}

/* ------------------------------------------------------------------ search */

struct ora_list {
    int n_sci, n_cj, n_pool;
    nbx_sci_entry* sci;
    nbx_cj_entry* cj;
    nbx_sci_entry* sci_in; /* inner ranges into cj_in (same offsets as outer) */
    nbx_cj_entry* cj_in;
    nbx_mask_pool_entry* pool;
    int mode;
};

static inline void shift_of(int s, int* sx, int* sy, int* sz)
{
    *sx = s % 3 - 1;
    *sy = (s / 3) % 3 - 1;
    *sz = s / 9 - 1;
}

static inline void shift_vec(int s, const float box[3], float v[3])
{
    int sx, sy, sz;
    shift_of(s, &sx, &sy, &sz);
    v[0] = (float)sx * box[0];
    v[1] = (float)sy * box[1];
    v[2] = (float)sz * box[2];
}

/* bounding-box distance^2 (a shifted by v), pinned operation order */
static inline float bb_dist2(const float* a, const float* v, const float* b)
{
    float d[3];
    for (int k = 0; k < 3; k++) {
        float alo = a[k] + v[k], ahi = a[3 + k] + v[k];
        float t = fmaxf(alo - b[3 + k], b[k] - ahi);
        d[k] = fmaxf(0.0f, t);
    }
    return fmaf(d[2], d[2], fmaf(d[1], d[1], d[0] * d[0]));
}

static int is_excluded(const ora_grid* g, int ga, int gb)
{
    for (int e = g->excl_offsets[ga]; e < g->excl_offsets[ga + 1]; e++)
        if (g->excl_gids[e] == gb) return 1;
    return 0;
}

typedef struct {
    void* p;
    size_t n, cap, esz;
} vec;

static void* vec_push(vec* v)
{
    if (v->n == v->cap) {
        v->cap = v->cap ? 2 * v->cap : 1024;
        v->p = realloc(v->p, v->cap * v->esz);
    }
    return (char*)v->p + (v->n++) * v->esz;
}

ora_list* ora_search(const ora_grid* gi, const ora_grid* gj, int mode, const nbx_params* p,
                     const float box[3], const int pbc[3])
{
    nbx_consts c;
    ora_derive_consts(p, &c);
    const float rl = p->rlist_outer, rl2 = c.rlo2;
    const float rlm = rl * 1.001f + 1.0e-4f;
    vec vs = {0, 0, 0, sizeof(nbx_sci_entry)};
    vec vc = {0, 0, 0, sizeof(nbx_cj_entry)};
    vec vp = {0, 0, 0, sizeof(nbx_mask_pool_entry)};
    nbx_mask_pool_entry* p0 = (nbx_mask_pool_entry*)vec_push(&vp);
    memset(p0, 0, sizeof(*p0));
    for (int k = 0; k < 8; k++) p0->m[k][0] = 0xffffffffu;

    for (int sci = 0; sci < gi->nsci; sci++) {
        if (gi->nreal_sci[sci] == 0) continue;
        for (int s = 0; s < NBX_NSHIFT; s++) {
            int sx, sy, sz;
            shift_of(s, &sx, &sy, &sz);
            if ((!pbc[0] && sx) || (!pbc[1] && sy) || (!pbc[2] && sz)) continue;
            if (mode == NBX_LIST_LOCAL && s < NBX_CENTRAL_SHIFT) continue;
            const int central = (s == NBX_CENTRAL_SHIFT);
            float v[3];
            shift_vec(s, box, v);
            const float* sb = gi->bb_sci + 6 * sci;
            float slo[3], shi[3];
            for (int d = 0; d < 3; d++) { slo[d] = sb[d] + v[d]; shi[d] = sb[3 + d] + v[d]; }
            int cx0 = (int)floorf((slo[0] - rl - gj->lo[0]) * gj->inv_cell[0]) - 1;
            int cx1 = (int)floorf((shi[0] + rl - gj->lo[0]) * gj->inv_cell[0]) + 1;
            int cy0 = (int)floorf((slo[1] - rl - gj->lo[1]) * gj->inv_cell[1]) - 1;
            int cy1 = (int)floorf((shi[1] + rl - gj->lo[1]) * gj->inv_cell[1]) + 1;
            if (cx0 < 0) cx0 = 0;
            if (cy0 < 0) cy0 = 0;
            if (cx1 > gj->ncx - 1) cx1 = gj->ncx - 1;
            if (cy1 > gj->ncy - 1) cy1 = gj->ncy - 1;
            int start = (int)vc.n;
            for (int cx = cx0; cx <= cx1; cx++) {
                for (int cy = cy0; cy <= cy1; cy++) {
                    int col = cx * gj->ncy + cy;
                    int k0 = gj->col_start[col] / 32, k1 = gj->col_start[col + 1] / 32;
                    for (int k = k0; k < k1; k++) {
                        const float* kb = gj->bb_sci + 6 * k;
                        if (kb[5] < slo[2] - rlm) continue;
                        if (kb[2] > shi[2] + rlm) break;
                        for (int cj = 4 * k; cj < 4 * k + 4; cj++) {
                            if (mode == NBX_LIST_LOCAL && central && cj < 4 * sci) continue;
                            if (gj->nreal_cj[cj] == 0) continue;
                            const float* bj = gj->bb_cj + 6 * cj;
                            if (!(bb_dist2(sb, v, bj) < rl2)) continue;
                            unsigned imask = 0;
                            int need_pool = 0;
                            uint32_t masks[8][2];
                            memset(masks, 0, sizeof(masks));
                            for (int kk = 0; kk < 8; kk++) {
                                int ci = 8 * sci + kk;
                                if (gi->nreal_ci[ci] == 0) continue;
                                if (!(bb_dist2(gi->bb_ci + 6 * ci, v, bj) < rl2)) continue;
                                int exov = !(gi->exhi_ci[ci] < gj->glo_cj[cj] || gi->exlo_ci[ci] > gj->ghi_cj[cj]);
                                int masked = gi->nreal_ci[ci] < 4 || gj->nreal_cj[cj] < 8 ||
                                             (central && (cj >> 2) == sci) || exov;
                                uint32_t im = 0xffffffffu, cm = 0u;
                                if (masked) {
                                    im = 0u;
                                    for (int i = 0; i < 4; i++) {
                                        int a = 4 * ci + i;
                                        if (gi->order[a] < 0) continue;
                                        int ga = gi->gid[a];
                                        for (int j = 0; j < 8; j++) {
                                            int b = 8 * cj + j;
                                            if (gj->order[b] < 0) continue;
                                            int gb = gj->gid[b];
                                            int present = (mode == NBX_LIST_LOCAL) ? !(central && b <= a) : 1;
                                            if (!present) continue;
                                            uint32_t bit = 1u << (i * 8 + j);
                                            if (exov && is_excluded(gi, ga, gb)) cm |= bit; else im |= bit;
                                        }
                                    }
                                    if ((im | cm) == 0u) continue;
                                }
                                imask |= 1u << kk;
                                masks[kk][0] = im;
                                masks[kk][1] = cm;
                                if (im != 0xffffffffu || cm != 0u) need_pool = 1;
                            }
                            if (!imask) continue;
                            uint32_t pidx = 0;
                            if (need_pool) {
                                pidx = (uint32_t)vp.n;
                                nbx_mask_pool_entry* pe = (nbx_mask_pool_entry*)vec_push(&vp);
                                for (int kk = 0; kk < 8; kk++) {
                                    pe->m[kk][0] = (imask >> kk & 1) ? masks[kk][0] : 0u;
                                    pe->m[kk][1] = (imask >> kk & 1) ? masks[kk][1] : 0u;
                                }
                            }
                            nbx_cj_entry* ce = (nbx_cj_entry*)vec_push(&vc);
                            ce->cj = cj;
                            ce->meta = imask | (pidx << 8);
                        }
                    }
                }
            }
            if ((int)vc.n > start) {
                nbx_sci_entry* se = (nbx_sci_entry*)vec_push(&vs);
                se->sci = sci;
                se->shift = s;
                se->cj_start = start;
                se->cj_end = (int)vc.n;
            }
        }
    }
    ora_list* l = (ora_list*)calloc(1, sizeof(ora_list));
    l->mode = mode;
    l->n_sci = (int)vs.n;
    l->n_cj = (int)vc.n;
    l->n_pool = (int)vp.n;
    l->sci = (nbx_sci_entry*)vs.p;
    l->cj = (nbx_cj_entry*)vc.p;
    l->pool = (nbx_mask_pool_entry*)vp.p;
    l->sci_in = (nbx_sci_entry*)malloc(sizeof(nbx_sci_entry) * (size_t)(l->n_sci + 1));
    l->cj_in = (nbx_cj_entry*)malloc(sizeof(nbx_cj_entry) * (size_t)(l->n_cj + 1));
    ora_prune(l, gi, gj, p, box, 0, 1);
    return l;
}

void ora_list_free(ora_list* l)
{
    if (!l) return;
    free(l->sci); free(l->cj); free(l->pool); free(l->sci_in); free(l->cj_in); free(l);
}

void ora_prune(ora_list* l, const ora_grid* gi, const ora_grid* gj, const nbx_params* p,
               const float box[3], int part, int nparts)
{
    nbx_consts c;
    ora_derive_consts(p, &c);
    const float rli2 = c.rli2;
#pragma omp parallel for schedule(dynamic, 16)
    for (int e = 0; e < l->n_sci; e++) {
        if (e % nparts != part) continue;
        const nbx_sci_entry se = l->sci[e];
        float v[3];
        shift_vec(se.shift, box, v);
        int kept = 0;
        for (int q = se.cj_start; q < se.cj_end; q++) {
            int cj = l->cj[q].cj;
            uint32_t meta = l->cj[q].meta, imask = meta & 0xffu, pidx = meta >> 8, nm = 0;
            for (int kk = 0; kk < 8; kk++) {
                if (!(imask >> kk & 1)) continue;
                uint32_t pm = l->pool[pidx].m[kk][0] | l->pool[pidx].m[kk][1];
                int ci = 8 * se.sci + kk, hit = 0;
                for (int i = 0; i < 4 && !hit; i++) {
                    const float* xa = gi->xq + 4 * (4 * ci + i);
                    float xs = xa[0] + v[0], ys = xa[1] + v[1], zs = xa[2] + v[2];
                    for (int j = 0; j < 8; j++) {
                        if (!(pm >> (i * 8 + j) & 1)) continue;
                        const float* xb = gj->xq + 4 * (8 * cj + j);
                        float dx = xs - xb[0], dy = ys - xb[1], dz = zs - xb[2];
                        float r2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
                        if (r2 < rli2) { hit = 1; break; }
                    }
                }
                if (hit) nm |= 1u << kk;
            }
            if (nm) {
                l->cj_in[se.cj_start + kept].cj = cj;
                l->cj_in[se.cj_start + kept].meta = nm | (pidx << 8);
                kept++;
            }
        }
        l->sci_in[e] = se;
        l->sci_in[e].cj_end = se.cj_start + kept;
    }
}

void ora_list_sizes(const ora_list* l, nbx_list_sizes* out)
{
    out->n_sci = l->n_sci;
    out->n_cj_outer = l->n_cj;
    int64_t in = 0;
    for (int e = 0; e < l->n_sci; e++) in += l->sci_in[e].cj_end - l->sci_in[e].cj_start;
    out->n_cj_inner = in;
    out->n_pool = l->n_pool;
}

void ora_list_export(const ora_list* l, int which, nbx_sci_entry* sci, nbx_cj_entry* cj,
                     nbx_mask_pool_entry* pool)
{
    if (pool) memcpy(pool, l->pool, sizeof(nbx_mask_pool_entry) * (size_t)l->n_pool);
    if (which == 0) {
        if (sci) memcpy(sci, l->sci, sizeof(nbx_sci_entry) * (size_t)l->n_sci);
        if (cj) memcpy(cj, l->cj, sizeof(nbx_cj_entry) * (size_t)l->n_cj);
        return;
    }
    int pos = 0;
    for (int e = 0; e < l->n_sci; e++) {
        nbx_sci_entry se = l->sci_in[e];
        int n = se.cj_end - se.cj_start;
        if (cj) memcpy(cj + pos, l->cj_in + se.cj_start, sizeof(nbx_cj_entry) * (size_t)n);
        if (sci) { sci[e] = se; sci[e].cj_start = pos; sci[e].cj_end = pos + n; }
        pos += n;
    }
}

/* ------------------------------------------------------------------ force */

typedef struct {
    float fscal, vlj, vc;
    int valid;
} pairres;

/* One atom pair: masked tiles carry explicit interaction (intb) and
 * exclusion-correction (corrb) bits, unmasked tiles have intb = 1, corrb = 0. */
static inline pairres pair_eval(float dx, float dy, float dz, int masked, int intb, int corrb,
                                float qi, float qj, float c6, float c12, const nbx_consts* c,
                                int coul, int energy, int ljmod, const float* ftab, const float* vtab)
{
    pairres r = {0.0f, 0.0f, 0.0f, 0};
    float r2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
    int valid = (r2 < c->rc2) && (masked ? (intb | corrb) : 1);
    if (!valid) return r;
    r.valid = 1;
    if (masked) r2 = fmaxf(r2, R2MIN);
    float rinv = 1.0f / sqrtf(r2);
    float rinv2 = rinv * rinv;
    float rinv3 = rinv * rinv2;
    float rinv6 = rinv3 * rinv3;
    float fint = masked ? (float)intb : 1.0f;
    float flj = (rinv6 * fmaf(c12, rinv6, -c6)) * fint;
    float qq = qi * qj;
    float fc, z = 0.0f;
    if (coul == NBX_COULOMB_RF) {
        fc = qq * fmaf(fint, rinv3, -(c->k_rf * 2.0f));
    } else if (coul == NBX_COULOMB_EWALD_TAB) {
        fc = qq * (fint * rinv3 - tab_interp(ftab, r2, rinv, c));
    } else {
        float beta2 = c->beta * c->beta;
        z = beta2 * r2;
        float G = ora_ewald_G(z);
        fc = qq * fmaf(-(beta2 * c->beta), G, fint * rinv3);
    }
    float rsw = 0.0f, rsw2 = 0.0f;
    if (ljmod == NBX_LJ_FORCE_SWITCH) {
        /* force switch on [r1, rc): F_a += A_a (r-r1)^2 + B_a (r-r1)^3 */
        float rr = r2 * rinv;
        rsw = fmaxf(rr - c->fsw_r1, 0.0f);
        rsw2 = rsw * rsw;
        float u = fmaf(c12, fmaf(c->fsw_b12, rsw, c->fsw_a12), -(c6 * fmaf(c->fsw_b6, rsw, c->fsw_a6)));
        fc = fc + ((u * rsw2) * rinv) * fint;
    }
    r.fscal = fmaf(flj, rinv2, fc);
    if (energy) {
        const float one6 = 1.0f / 6.0f, one12 = 1.0f / 12.0f;
        float vlj;
        if (ljmod == NBX_LJ_FORCE_SWITCH) {
            float rsw3 = rsw2 * rsw;
            float v12 = fmaf(rinv6, rinv6, -(fmaf(c->fsw_q12, rsw, c->fsw_p12) * rsw3)) - c->fsw_c12;
            float v6 = (rinv6 - fmaf(c->fsw_q6, rsw, c->fsw_p6) * rsw3) - c->fsw_c6;
            vlj = fmaf(c12 * one12, v12, -(c6 * one6) * v6);
        } else {
            vlj = fmaf(c12 * one12, fmaf(rinv6, rinv6, -c->sh_lj12), -(c6 * one6) * (rinv6 - c->sh_lj6));
        }
        r.vlj = vlj * fint;
        if (coul == NBX_COULOMB_RF)
            r.vc = qq * fmaf(c->k_rf, r2, fmaf(fint, rinv, -c->c_rf));
        else if (coul == NBX_COULOMB_EWALD_TAB)
            r.vc = qq * fmaf(fint, rinv - c->sh_ewald, -tab_interp(vtab, r2, rinv, c));
        else
            r.vc = qq * fmaf(fint, rinv - c->sh_ewald, -(c->beta * ora_ewald_H(z)));
    }
    return r;
}

/* LJ combination rules (nbx.h NBX_LJ_COMB_*): per-type parameters from the table diagonal,
 * in double, rounded once; zero for other modifiers.  Rule violations are not checked here
 * (the library's nbx_set_topology rejects them). */
void ora_lj_comb_params(int ljmod, int ntypes, const float* c6c12, float* pt)
{
    for (int a = 0; a < ntypes; a++) {
        const double c6 = c6c12[2 * (a * ntypes + a)], c12 = c6c12[2 * (a * ntypes + a) + 1];
        pt[2 * a] = pt[2 * a + 1] = 0.0f;
        if (ljmod == NBX_LJ_COMB_GEOM) {
            pt[2 * a] = (float)sqrt(6.0 * c6);
            pt[2 * a + 1] = (float)sqrt(12.0 * c12);
        } else if (ljmod == NBX_LJ_COMB_LB && c6 > 0.0 && c12 > 0.0) {
            const double sig = sqrt(cbrt(c12 / c6)), eps = c6 * c6 / (4.0 * c12);
            pt[2 * a] = (float)(0.5 * sig);
            pt[2 * a + 1] = (float)sqrt(24.0 * eps);
        }
    }
}

/* (6 c6, 12 c12) of a type pair: table lookup, or the combination rule in fp32 */
static inline void lj_pair(int ljmod, const float* pt, const float* c6c12, int ntypes, int ti, int tj,
                           float* c6, float* c12)
{
    if (ljmod == NBX_LJ_COMB_GEOM) {
        *c6 = pt[2 * ti] * pt[2 * tj];
        *c12 = pt[2 * ti + 1] * pt[2 * tj + 1];
    } else if (ljmod == NBX_LJ_COMB_LB) {
        const float sg = pt[2 * ti] + pt[2 * tj], s2 = sg * sg, s6 = (s2 * s2) * s2;
        const float p6 = (pt[2 * ti + 1] * pt[2 * tj + 1]) * s6;
        *c6 = p6;
        *c12 = 2.0f * (p6 * s6);
    } else {
        const float* cc = c6c12 + 2 * (ti * ntypes + tj);
        *c6 = 6.0f * cc[0];
        *c12 = 12.0f * cc[1];
    }
}

void ora_force(int n_sci, const nbx_sci_entry* sci, const nbx_cj_entry* cj,
               const nbx_mask_pool_entry* pool, const float* xq_i, const int* type_i,
               const float* xq_j, const int* type_j, int ntypes, const float* c6c12,
               const nbx_params* p, const float box[3], unsigned flags, double* f_i,
               double* f_j, double* e2, double* fshift, int nthreads)
{
    nbx_consts c;
    ora_derive_consts(p, &c);
    const int coul = p->coulomb_type, energy = (flags & NBX_FORCE_ENERGY) != 0, ljmod = p->lj_modifier;
    float* ptype = (float*)malloc(sizeof(float) * 2 * (size_t)ntypes);
    ora_lj_comb_params(ljmod, ntypes, c6c12, ptype);
    float* ftab = NULL;
    float* vtab = NULL;
    if (coul == NBX_COULOMB_EWALD_TAB) {
        ftab = (float*)malloc(sizeof(float) * 2 * (size_t)c.tab_n);
        vtab = (float*)malloc(sizeof(float) * 2 * (size_t)c.tab_n);
        ora_ewald_table(&c, ftab, vtab);
    }
    double elj = 0.0, ec = 0.0;
    double fsh[NBX_NSHIFT * 3];
    memset(fsh, 0, sizeof(fsh));
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#else
    nthreads = 1;
#endif
    /* Each thread accumulates into private force arrays only when running in parallel;
     * a serial run accumulates in place (j atoms of other entries make atomics necessary
     * otherwise).  Threads reduce in a fixed order, so results are deterministic for a
     * given thread count. */
    if (nthreads <= 1) {
        for (int e = 0; e < n_sci; e++) {
            nbx_sci_entry se = sci[e];
            float v[3];
            shift_vec(se.shift, box, v);
            for (int q = se.cj_start; q < se.cj_end; q++) {
                int cjj = cj[q].cj;
                uint32_t meta = cj[q].meta, imask = meta & 0xffu, pidx = meta >> 8;
                int masked = pidx != 0;
                for (int kk = 0; kk < 8; kk++) {
                    if (!(imask >> kk & 1)) continue;
                    uint32_t im = pool[pidx].m[kk][0], cm = pool[pidx].m[kk][1];
                    if (!masked) { im = 0xffffffffu; cm = 0u; }
                    int ci = 8 * se.sci + kk;
                    for (int i = 0; i < 4; i++) {
                        int a = 4 * ci + i;
                        const float* xa = xq_i + 4 * a;
                        float xs = xa[0] + v[0], ys = xa[1] + v[1], zs = xa[2] + v[2];
                        float qi = xa[3] * c.epsfac;
                        int ti = type_i[a];
                        for (int j = 0; j < 8; j++) {
                            int b = 8 * cjj + j;
                            const float* xb = xq_j + 4 * b;
                            float dx = xs - xb[0], dy = ys - xb[1], dz = zs - xb[2];
                            int bit = i * 8 + j;
                            float c6, c12;
                            lj_pair(ljmod, ptype, c6c12, ntypes, ti, type_j[b], &c6, &c12);
                            pairres r = pair_eval(dx, dy, dz, masked, (im >> bit) & 1, (cm >> bit) & 1,
                                                  qi, xb[3], c6, c12, &c, coul, energy, ljmod, ftab, vtab);
                            if (!r.valid) continue;
                            float fx = r.fscal * dx, fy = r.fscal * dy, fz = r.fscal * dz;
                            f_i[3 * a + 0] += fx; f_i[3 * a + 1] += fy; f_i[3 * a + 2] += fz;
                            f_j[3 * b + 0] -= fx; f_j[3 * b + 1] -= fy; f_j[3 * b + 2] -= fz;
                            fsh[3 * se.shift + 0] += fx; fsh[3 * se.shift + 1] += fy; fsh[3 * se.shift + 2] += fz;
                            if (energy) { elj += r.vlj; ec += r.vc; }
                        }
                    }
                }
            }
        }
    } else {
        /* parallel: thread-private force buffers (i and j; one buffer when they alias),
         * reduced in thread order afterwards */
        int maxi = 0, maxj = 0;
        for (int e = 0; e < n_sci; e++) {
            if (32 * sci[e].sci + 32 > maxi) maxi = 32 * sci[e].sci + 32;
            for (int q = sci[e].cj_start; q < sci[e].cj_end; q++)
                if (8 * cj[q].cj + 8 > maxj) maxj = 8 * cj[q].cj + 8;
        }
        const int same = (f_i == f_j);
        const int nbj = same ? (maxi > maxj ? maxi : maxj) : maxj;
        const int nbi = same ? 0 : maxi;
        const size_t per = (size_t)(nbj + nbi) * 3;
        double* priv = (double*)calloc((size_t)nthreads * per, sizeof(double));
        double* pe = (double*)calloc((size_t)nthreads * (2 + 3 * NBX_NSHIFT), sizeof(double));
#pragma omp parallel num_threads(nthreads)
        {
            int t = 0;
#ifdef _OPENMP
            t = omp_get_thread_num();
#endif
            double* fj = priv + (size_t)t * per;
            double* fi = same ? fj : fj + (size_t)nbj * 3;
            double* my = pe + (size_t)t * (2 + 3 * NBX_NSHIFT);
#pragma omp for schedule(dynamic, 4)
            for (int e = 0; e < n_sci; e++) {
                nbx_sci_entry se = sci[e];
                float v[3];
                shift_vec(se.shift, box, v);
                double fiacc[32][3];
                memset(fiacc, 0, sizeof(fiacc));
                for (int q = se.cj_start; q < se.cj_end; q++) {
                    int cjj = cj[q].cj;
                    uint32_t meta = cj[q].meta, imask = meta & 0xffu, pidx = meta >> 8;
                    int masked = pidx != 0;
                    for (int kk = 0; kk < 8; kk++) {
                        if (!(imask >> kk & 1)) continue;
                        uint32_t im = pool[pidx].m[kk][0], cm = pool[pidx].m[kk][1];
                        if (!masked) { im = 0xffffffffu; cm = 0u; }
                        int ci = 8 * se.sci + kk;
                        for (int i = 0; i < 4; i++) {
                            int a = 4 * ci + i;
                            const float* xa = xq_i + 4 * a;
                            float xs = xa[0] + v[0], ys = xa[1] + v[1], zs = xa[2] + v[2];
                            float qi = xa[3] * c.epsfac;
                            int ti = type_i[a];
                            for (int j = 0; j < 8; j++) {
                                int b = 8 * cjj + j;
                                const float* xb = xq_j + 4 * b;
                                float dx = xs - xb[0], dy = ys - xb[1], dz = zs - xb[2];
                                int bit = i * 8 + j;
                                float c6, c12;
                                lj_pair(ljmod, ptype, c6c12, ntypes, ti, type_j[b], &c6, &c12);
                                pairres r = pair_eval(dx, dy, dz, masked, (im >> bit) & 1, (cm >> bit) & 1,
                                                      qi, xb[3], c6, c12, &c, coul, energy, ljmod, ftab, vtab);
                                if (!r.valid) continue;
                                float fx = r.fscal * dx, fy = r.fscal * dy, fz = r.fscal * dz;
                                fiacc[a - 32 * se.sci][0] += fx;
                                fiacc[a - 32 * se.sci][1] += fy;
                                fiacc[a - 32 * se.sci][2] += fz;
                                fj[3 * b + 0] -= fx; fj[3 * b + 1] -= fy; fj[3 * b + 2] -= fz;
                                if (energy) { my[0] += r.vlj; my[1] += r.vc; }
                            }
                        }
                    }
                }
                for (int a = 0; a < 32; a++)
                    for (int d = 0; d < 3; d++) {
                        fi[3 * (32 * se.sci + a) + d] += fiacc[a][d];
                        my[2 + 3 * se.shift + d] += fiacc[a][d];
                    }
            }
        }
        for (int t = 0; t < nthreads; t++) {
            double* fj = priv + (size_t)t * per;
            for (int k = 0; k < 3 * nbj; k++) f_j[k] += fj[k];
            if (!same) for (int k = 0; k < 3 * nbi; k++) f_i[k] += fj[3 * nbj + k];
            double* my = pe + (size_t)t * (2 + 3 * NBX_NSHIFT);
            elj += my[0];
            ec += my[1];
            for (int k = 0; k < 3 * NBX_NSHIFT; k++) fsh[k] += my[2 + k];
        }
        free(priv);
        free(pe);
    }
    if (e2) { e2[0] += elj; e2[1] += ec; }
    if (fshift) for (int k = 0; k < 3 * NBX_NSHIFT; k++) fshift[k] += fsh[k];
    free(ptype);
    free(ftab);
    free(vtab);
}

long long ora_count_pairs(int n_sci, const nbx_sci_entry* sci, const nbx_cj_entry* cj,
                          const nbx_mask_pool_entry* pool, const float* xq_i, const float* xq_j,
                          const nbx_params* p, const float box[3])
{
    nbx_consts c;
    ora_derive_consts(p, &c);
    long long n = 0;
#pragma omp parallel for reduction(+ : n) schedule(dynamic, 16)
    for (int e = 0; e < n_sci; e++) {
        float v[3];
        shift_vec(sci[e].shift, box, v);
        for (int q = sci[e].cj_start; q < sci[e].cj_end; q++) {
            uint32_t meta = cj[q].meta, imask = meta & 0xffu, pidx = meta >> 8;
            for (int kk = 0; kk < 8; kk++) {
                if (!(imask >> kk & 1)) continue;
                uint32_t im = pidx ? pool[pidx].m[kk][0] : 0xffffffffu;
                for (int i = 0; i < 4; i++) {
                    const float* xa = xq_i + 4 * (4 * (8 * sci[e].sci + kk) + i);
                    float xs = xa[0] + v[0], ys = xa[1] + v[1], zs = xa[2] + v[2];
                    for (int j = 0; j < 8; j++) {
                        if (!(im >> (i * 8 + j) & 1)) continue;
                        const float* xb = xq_j + 4 * (8 * cj[q].cj + j);
                        float dx = xs - xb[0], dy = ys - xb[1], dz = zs - xb[2];
                        if (fmaf(dz, dz, fmaf(dy, dy, dx * dx)) < c.rc2) n++;
                    }
                }
            }
        }
    }
    return n;
}

void ora_virial(const ora_grid* g, const double* f_slots, const double* fshift,
                const float box[3], double* vir)
{
    double w[9] = {0};
    for (int s = 0; s < g->nslots; s++) {
        if (g->order[s] < 0) continue;
        for (int a = 0; a < 3; a++)
            for (int b = 0; b < 3; b++) w[3 * a + b] += (double)g->xq[4 * s + a] * f_slots[3 * s + b];
    }
    if (fshift) {
        for (int s = 0; s < NBX_NSHIFT; s++) {
            float v[3];
            shift_vec(s, box, v);
            for (int a = 0; a < 3; a++)
                for (int b = 0; b < 3; b++) w[3 * a + b] += (double)v[a] * fshift[3 * s + b];
        }
    }
    for (int k = 0; k < 9; k++) vir[k] = -0.5 * w[k];
}
