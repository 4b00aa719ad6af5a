/* nbx_c_smoke.c -- a plain C99 consumer of the C-ABI (include/nbx.h), the way an integrator
 * without Python would bind libnbx.so.  Builds a small SPC/E-like
 * water lattice, runs the reference cadence for a few steps with Ewald + PME + leap-frog, and
 * checks the results the physics guarantees without an oracle:
 *   - every call returns NBX_OK;
 *   - nonbonded forces are finite and sum to ~0 (Newton's third law over the half list);
 *   - the energy step reproduces the force-only step's forces;
 *   - an invalid call fails with NBX_EINVAL and a message (no silent fallback).
 * Prints "nbx_c_smoke ok ..." and exits 0 on success.  Built by tests/test_c_abi.py with gcc
 * against include/nbx.h and libnbx.so; the device buffers come from the CUDA runtime API.  */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime_api.h>

#include "nbx.h"

#define CHECK(call)                                                                         \
    do {                                                                                    \
        int rc_ = (call);                                                                   \
        if (rc_ != NBX_OK) {                                                                \
            fprintf(stderr, "%s failed (%d): %s\n", #call, rc_, nbx_last_error());          \
            return 1;                                                                       \
        }                                                                                   \
    } while (0)

#define CUDA(call)                                                                          \
    do {                                                                                    \
        cudaError_t e_ = (call);                                                            \
        if (e_ != cudaSuccess) {                                                            \
            fprintf(stderr, "%s failed: %s\n", #call, cudaGetErrorString(e_));              \
            return 1;                                                                       \
        }                                                                                   \
    } while (0)

static double urand(unsigned* s)
{
    *s = *s * 1664525u + 1013904223u;
    return (double)(*s >> 8) / 16777216.0;
}

int main(void)
{
    const int nside = 12, nmol = nside * nside * nside, n = 3 * nmol;
    const float spacing = 0.3107f, L = nside * spacing;
    float* x = malloc(sizeof(float) * 3 * n);
    float* q = malloc(sizeof(float) * n);
    int32_t* type = malloc(sizeof(int32_t) * n);
    int32_t* eoff = malloc(sizeof(int32_t) * (n + 1));
    int32_t* egid = malloc(sizeof(int32_t) * 2 * n);
    unsigned seed = 12345u;
    int ne = 0;
    for (int m = 0; m < nmol; m++) {
        const int a = m % nside, b = (m / nside) % nside, c = m / (nside * nside);
        const float o[3] = {(a + 0.5f) * spacing, (b + 0.5f) * spacing, (c + 0.5f) * spacing};
        for (int k = 0; k < 3; k++) {
            const int id = 3 * m + k;
            for (int d = 0; d < 3; d++)
                x[3 * id + d] = o[d] + (k ? 0.1f * (float)(urand(&seed) - 0.5) * 2.0f : 0.0f);
            q[id] = k ? 0.4238f : -0.8476f;
            type[id] = k ? 1 : 0;
        }
    }
    for (int id = 0; id < n; id++) { /* intramolecular exclusions: the other two atoms */
        const int m = id / 3;
        eoff[id] = ne;
        for (int k = 0; k < 3; k++)
            if (3 * m + k != id) egid[ne++] = 3 * m + k;
    }
    eoff[n] = ne;
    const double sig = 0.316557, eps = 0.650194;
    const float c6c12[2 * 2 * 2] = {(float)(4 * eps * pow(sig, 6)), (float)(4 * eps * pow(sig, 12)), 0, 0, 0, 0, 0, 0};

    nbx_params p;
    memset(&p, 0, sizeof(p));
    p.coulomb_type = NBX_COULOMB_EWALD;
    p.rc = 1.0f;
    p.rlist_outer = 1.1f;
    p.rlist_inner = 1.02f;
    p.epsilon_r = 1.0f;
    p.epsilon_rf = 0.0f;
    p.ewald_rtol = 1e-5f;
    p.lj_modifier = NBX_LJ_POT_SHIFT;
    nbx_consts c;
    CHECK(nbx_derive_consts(&p, &c));

    nbx_ctx* ctx = NULL;
    CHECK(nbx_create(0, &p, &ctx));
    CHECK(nbx_set_topology(ctx, n, q, type, 2, c6c12, eoff, egid));
    const float box[3] = {L, L, L}, lo[3] = {0, 0, 0};
    const int32_t pbc[3] = {1, 1, 1};
    CHECK(nbx_set_box(ctx, box, pbc));

    float *xd, *fd, *f2d, *qd, *vd, *imd;
    CUDA(cudaMalloc((void**)&xd, sizeof(float) * 3 * n));
    CUDA(cudaMalloc((void**)&fd, sizeof(float) * 3 * n));
    CUDA(cudaMalloc((void**)&f2d, sizeof(float) * 3 * n));
    CUDA(cudaMalloc((void**)&vd, sizeof(float) * 3 * n));
    CUDA(cudaMalloc((void**)&qd, sizeof(float) * n));
    CUDA(cudaMalloc((void**)&imd, sizeof(float) * n));
    CUDA(cudaMemcpy(xd, x, sizeof(float) * 3 * n, cudaMemcpyHostToDevice));
    CUDA(cudaMemcpy(qd, q, sizeof(float) * n, cudaMemcpyHostToDevice));
    CUDA(cudaMemset(vd, 0, sizeof(float) * 3 * n));
    float* im = malloc(sizeof(float) * n);
    for (int a = 0; a < n; a++) im[a] = 1.0f / (type[a] ? 1.008f : 15.999f);
    CUDA(cudaMemcpy(imd, im, sizeof(float) * n, cudaMemcpyHostToDevice));

    nbx_pme_params pp;
    const int K = 2 * (int)ceil(L / 0.12 / 2.0);
    pp.nk[0] = pp.nk[1] = pp.nk[2] = K < 8 ? 8 : K;
    pp.order = 4;
    pp.beta = c.beta;
    pp.epsfac = c.epsfac;
    nbx_pme* pme = NULL;
    CHECK(nbx_pme_create(0, &pp, &pme));
    CHECK(nbx_pme_set_box(pme, box));

    /* reference cadence (pipeline.py:222-235) with PME + update; dt = 0 keeps x fixed so the
     * force-only and energy steps below see identical coordinates */
    for (int step = 0; step < 12; step++) {
        if (step % 100 == 0) {
            CHECK(nbx_grid_build(ctx, 0, n, xd, NULL, lo, box, NULL));
            CHECK(nbx_search(ctx, NBX_LIST_LOCAL, NULL));
        } else {
            CHECK(nbx_put_x(ctx, 0, xd, NULL));
            if (step % 10 == 0) CHECK(nbx_prune(ctx, NBX_LIST_LOCAL, 0, 1, NULL));
        }
        CHECK(nbx_force(ctx, NBX_LIST_LOCAL, 0, NULL));
        CHECK(nbx_get_f(ctx, 0, fd, 0, NULL));
        CHECK(nbx_pme_compute(pme, n, xd, qd, fd, 0, NULL));
        CHECK(nbx_leapfrog(n, xd, vd, fd, imd, 0.0f, NULL));
    }
    /* nonbonded forces alone: force-only vs energy step */
    CHECK(nbx_put_x(ctx, 0, xd, NULL));
    CHECK(nbx_force(ctx, NBX_LIST_LOCAL, 0, NULL));
    CHECK(nbx_get_f(ctx, 0, fd, 0, NULL));
    CHECK(nbx_clear_energies(ctx, NULL));
    CHECK(nbx_force(ctx, NBX_LIST_LOCAL, NBX_FORCE_ENERGY | NBX_FORCE_VIRIAL, NULL));
    double e[2], vir[9];
    CHECK(nbx_energies(ctx, e, vir, NULL));
    CHECK(nbx_get_f(ctx, 0, f2d, 0, NULL));
    CHECK(nbx_pme_compute(pme, n, xd, qd, f2d, NBX_FORCE_ENERGY, NULL));
    double erec, vrec[9];
    CHECK(nbx_pme_energy(pme, &erec, vrec, NULL));
    CUDA(cudaDeviceSynchronize());

    float* f = malloc(sizeof(float) * 3 * n);
    float* f2 = malloc(sizeof(float) * 3 * n);
    CUDA(cudaMemcpy(f, fd, sizeof(float) * 3 * n, cudaMemcpyDeviceToHost));
    CUDA(cudaMemcpy(f2, f2d, sizeof(float) * 3 * n, cudaMemcpyDeviceToHost));
    double sum[3] = {0, 0, 0}, sq = 0.0, dd = 0.0;
    for (int a = 0; a < n; a++)
        for (int d = 0; d < 3; d++) {
            const double v = f[3 * a + d];
            if (!isfinite(v)) {
                fprintf(stderr, "non-finite force\n");
                return 1;
            }
            sum[d] += v;
            sq += v * v;
        }
    const double rms = sqrt(sq / (3.0 * n));
    if (fabs(sum[0]) + fabs(sum[1]) + fabs(sum[2]) > 1e-3 * rms * n) {
        fprintf(stderr, "Newton III violated: sum %g %g %g (rms %g)\n", sum[0], sum[1], sum[2], rms);
        return 1;
    }
    /* f2 = NB (energy kernel) + PME; f = NB (force-only): they differ by the PME forces only,
     * so compare NB + PME against NB + PME recomputed on the force-only forces */
    CHECK(nbx_pme_compute(pme, n, xd, qd, fd, 0, NULL));
    CUDA(cudaMemcpy(f, fd, sizeof(float) * 3 * n, cudaMemcpyDeviceToHost));
    for (int k = 0; k < 3 * n; k++) dd += (f[k] - f2[k]) * (double)(f[k] - f2[k]);
    if (sqrt(dd / (3.0 * n)) > 1e-5 * rms) {
        fprintf(stderr, "energy step forces differ: rms diff %g vs rms %g\n", sqrt(dd / (3.0 * n)), rms);
        return 1;
    }
    if (!isfinite(e[0]) || !(e[1] < 0.0) || !(erec > 0.0)) {
        fprintf(stderr, "implausible energies: E_lj %g E_coul %g E_rec %g\n", e[0], e[1], erec);
        return 1;
    }
    if (nbx_prune(ctx, NBX_LIST_LOCAL, 3, 2, NULL) != NBX_EINVAL || strlen(nbx_last_error()) == 0) {
        fprintf(stderr, "bad prune part did not fail with NBX_EINVAL\n");
        return 1;
    }
    printf("nbx_c_smoke ok: %d atoms, E_lj %.3f E_coul %.3f E_rec %.3f kJ/mol, |sum f| / rms %.2e, "
           "%lld + %lld launches\n",
           n, e[0], e[1], erec, (fabs(sum[0]) + fabs(sum[1]) + fabs(sum[2])) / rms, (long long)nbx_launch_count(ctx),
           (long long)nbx_pme_launch_count(pme));
    CHECK(nbx_pme_destroy(pme));
    CHECK(nbx_destroy(ctx));
    cudaFree(xd);
    cudaFree(fd);
    cudaFree(f2d);
    cudaFree(vd);
    cudaFree(qd);
    cudaFree(imd);
    free(x);
    free(q);
    free(type);
    free(eoff);
    free(egid);
    free(im);
    free(f);
    free(f2);
    return 0;
}
