// capi.cu -- the extern "C" boundary of libnbx.so (include/nbx.h).  Every entry point
// catches all errors and returns an nbx_status with a thread-local message; no exception
// crosses the ABI.  There is no CPU fallback anywhere in this library.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "nbx_internal.cuh"

namespace nbx {

static thread_local std::string g_err;
unsigned long long g_allocs = 0;
int g_trace_allocs = std::getenv("NBX_TRACE_ALLOCS") ? std::atoi(std::getenv("NBX_TRACE_ALLOCS")) : 0;

void trace_alloc(size_t bytes, size_t old_bytes, void* caller)
{
    std::fprintf(stderr, "[nbx alloc #%llu] %zu bytes (was %zu) from %p\n", g_allocs, bytes, old_bytes, caller);
}

void set_error(const std::string& msg) { g_err = msg; }

int fail(int code, const std::string& msg)
{
    g_err = msg;
    return code;
}

static double ewald_beta(double rc, double rtol)
{
    double lo = 0.0, hi = 5.0;
    while (std::erfc(hi * rc) > rtol) hi *= 2.0;
    for (int it = 0; it < 60; it++) {
        double mid = 0.5 * (lo + hi);
        if (std::erfc(mid * rc) > rtol) lo = mid; else hi = mid;
    }
    return 0.5 * (lo + hi);
}

// identical formulas to ora_derive_consts (oracle/nbx_oracle.c)
static int derive(const nbx_params* p, nbx_consts* c)
{
    const double rc = p->rc;
    std::memset(c, 0, sizeof(*c));
    c->epsfac = (float)(138.935458 / (double)p->epsilon_r);
    double krf;
    if (p->epsilon_rf == 0.0f)
        krf = 1.0 / (2.0 * rc * rc * rc);
    else
        krf = ((double)p->epsilon_rf - (double)p->epsilon_r) /
              ((2.0 * (double)p->epsilon_rf + (double)p->epsilon_r) * rc * rc * rc);
    c->k_rf = (float)krf;
    c->c_rf = (float)(1.0 / rc + krf * rc * rc);
    const bool ew = p->coulomb_type == NBX_COULOMB_EWALD || p->coulomb_type == NBX_COULOMB_EWALD_TAB;
    const double beta = ew ? ewald_beta(rc, p->ewald_rtol) : 0.0;
    c->beta = (float)beta;
    c->sh_ewald = ew ? (float)(std::erfc(beta * rc) / rc) : 0.0f;
    if (p->coulomb_type == NBX_COULOMB_EWALD_TAB) {
        c->tab_scale = (float)(400.0 * beta > 600.0 ? 400.0 * beta : 600.0);
        c->tab_n = (int32_t)std::ceil(rc * (double)c->tab_scale) + 2;
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
            const double a = al[k], rca2 = std::pow(rc, a + 2.0);
            A[k] = -a * ((a + 4.0) * rc - (a + 1.0) * r1) / (rca2 * d * d);
            B[k] = a * ((a + 3.0) * rc - (a + 1.0) * r1) / (rca2 * d * d * d);
            C[k] = std::pow(rc, -a) - A[k] / 3.0 * d * d * d - B[k] / 4.0 * d * d * d * d;
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
    if (p->lj_modifier < NBX_LJ_POT_SHIFT || p->lj_modifier > NBX_LJ_COMB_LB) return 1;
    if (p->lj_modifier == NBX_LJ_FORCE_SWITCH && !(p->rvdw_switch >= 0.0f && p->rvdw_switch < p->rc)) return 1;
    if (!(p->rc > 0.0f) || p->rlist_inner < p->rc || p->rlist_outer < p->rlist_inner) return 1;
    if (p->coulomb_type != NBX_COULOMB_RF && !ew) return 1;
    if (ew && !(p->ewald_rtol > 0.0f && p->ewald_rtol < 1.0f)) return 1;
    if (!(p->epsilon_r > 0.0f)) return 1;
    return 0;
}

// EWALD_TAB tables, identical formulas to ora_ewald_table (oracle/nbx_oracle.c): nodes
// r_k = k / tab_scale; force correction beta^3 G(beta^2 r^2) with its series below z = 1e-2,
// potential erf(beta r) / r; stored as (value, next - value)
static double ewald_fcorr(double beta, double r)
{
    const double z = beta * beta * r * r, b3 = beta * beta * beta, tsp = 2.0 / std::sqrt(M_PI);
    if (z < 1e-2) return tsp * b3 * (2.0 / 3.0 + z * (-2.0 / 5.0 + z * (1.0 / 7.0 + z * (-1.0 / 27.0 + z / 132.0))));
    return (std::erf(beta * r) / r - tsp * beta * std::exp(-z)) / (r * r);
}

static double ewald_vcorr(double beta, double r)
{
    if (r == 0.0) return 2.0 * beta / std::sqrt(M_PI);
    return std::erf(beta * r) / r;
}

int ewald_table(const nbx_consts* c, float* ftab, float* vtab)
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

} // namespace nbx

using namespace nbx;

#define NBX_GUARD_BEGIN try {
#define NBX_GUARD_END                                                                         \
    }                                                                                         \
    catch (const CudaError& e)                                                                \
    {                                                                                         \
        int code = (e.err == cudaErrorMemoryAllocation) ? NBX_ENOMEM : NBX_ECUDA;            \
        if (std::strstr(e.what, "24-bit")) code = NBX_ELIST_OVERFLOW;                        \
        return fail(code, std::string(e.what) + ": " + cudaGetErrorString(e.err));           \
    }                                                                                         \
    catch (const std::exception& e)                                                           \
    {                                                                                         \
        return fail(NBX_EINVAL, e.what());                                                    \
    }                                                                                         \
    catch (...)                                                                               \
    {                                                                                         \
        return fail(NBX_EINVAL, "unknown error");                                             \
    }

#define NBX_CHECK_CTX(ctx)                                                                    \
    if (!(ctx)) return fail(NBX_EINVAL, "null context");                                      \
    NBX_CUDA(cudaSetDevice((ctx)->device));

extern "C" {

NBX_API const char* nbx_last_error(void) { return g_err.c_str(); }

NBX_API const char* nbx_version(void) { return NBX_CHECKED ? "nbx 0.1 (sm_100a, checked)" : "nbx 0.1 (sm_100a)"; }

NBX_API int nbx_derive_consts(const nbx_params* p, nbx_consts* out)
{
    if (!p || !out) return fail(NBX_EINVAL, "null argument");
    if (derive(p, out)) return fail(NBX_EINVAL, "invalid parameters (need 0 < rc <= rlist_inner <= rlist_outer, valid coulomb type)");
    return NBX_OK;
}

NBX_API int nbx_ewald_table(const nbx_consts* c, float* ftab, float* vtab)
{
    if (!c || !ftab || !vtab) return fail(NBX_EINVAL, "null argument");
    if (ewald_table(c, ftab, vtab)) return fail(NBX_EINVAL, "constants carry no Ewald table (coulomb_type != EWALD_TAB)");
    return NBX_OK;
}

NBX_API int nbx_create(int device, const nbx_params* p, nbx_ctx** out)
{
    NBX_GUARD_BEGIN
    if (!p || !out) return fail(NBX_EINVAL, "null argument");
    *out = nullptr;
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev <= device || device < 0)
        return fail(NBX_ECUDA, std::string("no CUDA device ") + std::to_string(device) + " (" +
                                   cudaGetErrorString(e) + "); libnbx has no CPU fallback");
    cudaDeviceProp prop;
    NBX_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
        return fail(NBX_ECUDA, std::string("device ") + prop.name + " is not sm_100 (built for sm_100a only)");
    nbx_consts c;
    if (derive(p, &c)) return fail(NBX_EINVAL, "invalid parameters");
    NBX_CUDA(cudaSetDevice(device));
    nbx_ctx* ctx = new nbx_ctx();
    ctx->device = device;
    ctx->num_sms = prop.multiProcessorCount;
    ctx->p = *p;
    ctx->c = c;
    ctx->acc.ensure(2 + 3 * NBX_NSHIFT + 9);
    NBX_CUDA(cudaMemset(ctx->acc.p, 0, sizeof(double) * (2 + 3 * NBX_NSHIFT + 9)));
    if (p->coulomb_type == NBX_COULOMB_EWALD_TAB) {
        std::vector<float> ft(2 * (size_t)c.tab_n), vt(2 * (size_t)c.tab_n);
        ewald_table(&c, ft.data(), vt.data());
        ctx->ewtab.ensure(2 * (size_t)c.tab_n); // [tab_n] force pairs, then [tab_n] potential pairs
        NBX_CUDA(cudaMemcpy(ctx->ewtab.p, ft.data(), sizeof(float) * ft.size(), cudaMemcpyHostToDevice));
        NBX_CUDA(cudaMemcpy(ctx->ewtab.p + c.tab_n, vt.data(), sizeof(float) * vt.size(), cudaMemcpyHostToDevice));
    }
    ctx->sumq2.ensure(2);
    NBX_CUDA(cudaMemset(ctx->sumq2.p, 0, sizeof(double) * 2));
    ctx->counter.ensure(8);
    // Row f2 (list sorting by length): automatic by list size (entry_order = -1,
    // nbx_internal.cuh) -- on for the mid-size lists whose tail it shortens, off for the 12 M
    // box (longest-first costs L2 locality there, +5 %) and for tiny lists; DESIGN.md section 5
    if (const char* pk = std::getenv("NBX_PRUNE_KERNEL")) ctx->prune_kernel = std::atoi(pk);
    if (const char* ps = std::getenv("NBX_PRUNE_SPLIT")) ctx->prune_split = std::atoi(ps);
    if (const char* eo = std::getenv("NBX_ENTRY_ORDER")) ctx->entry_order = std::atoi(eo);
    if (const char* fs = std::getenv("NBX_FORCE_SPLIT")) ctx->force_split = std::atoi(fs);
    *out = ctx;
    return NBX_OK;
    NBX_GUARD_END
}

NBX_API int nbx_destroy(nbx_ctx* ctx)
{
    NBX_GUARD_BEGIN
    if (!ctx) return NBX_OK;
    cudaSetDevice(ctx->device);
    cudaDeviceSynchronize();
    for (int g = 0; g < 2; g++) {
        Grid& G = ctx->grid[g];
        G.col_count.release(); G.col_start.release(); G.col_astart.release();
        G.key.release(); G.key_out.release(); G.val.release(); G.val_out.release(); G.xw.release();
        G.order.release(); G.gid.release(); G.type.release(); G.xq.release(); G.wrapk.release();
        G.f.release(); G.bb_ci.release(); G.bb_cj.release(); G.bb_sci.release();
        G.slotmap.release(); G.islot.release(); G.bb_col.release(); G.tmp.release(); G.padded.release();
        List& L = ctx->list[g];
        L.sci.release(); L.sci_in.release(); L.cj.release(); L.cj_in.release(); L.pool.release();
        L.counts.release(); L.offsets.release(); L.totals.release(); L.tmp.release();
        L.len_key.release(); L.len_key_out.release(); L.order_in.release(); L.order.release(); L.sort_tmp.release();
        L.flags.release(); L.tsci.release(); L.tcj.release(); L.tpool.release(); L.pair_count.release();
        L.prune_tmp.release(); L.prune_kept.release();
    }
    ctx->q_g.release(); ctx->type_g.release(); ctx->excl_off_g.release(); ctx->excl_gid_g.release();
    ctx->c6c12s.release(); ctx->acc.release(); ctx->sumq2.release(); ctx->counter.release();
    ctx->ewtab.release();
    for (auto& g : ctx->graphs) cudaGraphExecDestroy(g.exec);
    for (auto& g : ctx->full_graphs) cudaGraphExecDestroy(g.exec);
    peer_release(ctx);
    if (ctx->cap_stream) cudaStreamDestroy(ctx->cap_stream);
    if (ctx->h_pin) cudaFreeHost(ctx->h_pin);
    for (cudaEvent_t e : ctx->ev_pair)
        if (e) cudaEventDestroy(e);
    delete ctx;
    return NBX_OK;
    NBX_GUARD_END
}

NBX_API int nbx_set_topology(nbx_ctx* ctx, int32_t n, const float* q, const int32_t* type,
                             int32_t ntypes, const float* c6c12, const int32_t* excl_offsets,
                             const int32_t* excl_gids)
{
    NBX_GUARD_BEGIN
    NBX_CHECK_CTX(ctx);
    if (n < 0 || ntypes <= 0 || !q || !type || !c6c12 || !excl_offsets)
        return fail(NBX_EINVAL, "bad topology arguments");
    if ((size_t)ntypes * ntypes * sizeof(float2) > 48 * 1024)
        return fail(NBX_EINVAL, "too many LJ types for the shared-memory table (max 78)");
    for (int a = 0; a < n; a++)
        if (type[a] < 0 || type[a] >= ntypes) return fail(NBX_EINVAL, "atom type out of range");
    {
        // force kernel shared memory: the LJ table (+ the EWALD_TAB force and potential tables)
        const bool comb = ctx->p.lj_modifier == NBX_LJ_COMB_GEOM || ctx->p.lj_modifier == NBX_LJ_COMB_LB;
        const size_t tab = ctx->p.coulomb_type == NBX_COULOMB_EWALD_TAB ? 2 * (size_t)ctx->c.tab_n : 0;
        if (((comb ? (size_t)ntypes : (size_t)ntypes * ntypes) + tab) * sizeof(float2) > FORCE_SMEM_MAX)
            return fail(NBX_EINVAL, "LJ + Ewald tables exceed the force kernel's shared-memory opt-in");
    }
    const int nexcl = excl_offsets[n];
    if (excl_offsets[0] != 0 || nexcl < 0 || (nexcl > 0 && !excl_gids))
        return fail(NBX_EINVAL, "bad exclusion CSR");
    // offsets monotone and inside [0, nexcl] (the search's mask builder walks them unchecked)
    for (int a = 0; a < n; a++)
        if (excl_offsets[a] > excl_offsets[a + 1] || excl_offsets[a + 1] > nexcl)
            return fail(NBX_EINVAL, "exclusion CSR offsets are not monotone / exceed the id count");
    for (int e = 0; e < nexcl; e++)
        if (excl_gids[e] < 0 || excl_gids[e] >= n) return fail(NBX_EINVAL, "exclusion id out of range");
    // symmetry: b in excl(a) <=> a in excl(b); otherwise a tile's masks would depend on which
    // atom of the pair lands in the i-cluster
    for (int a = 0; a < n; a++)
        for (int e = excl_offsets[a]; e < excl_offsets[a + 1]; e++) {
            const int b = excl_gids[e];
            bool found = false;
            for (int k = excl_offsets[b]; k < excl_offsets[b + 1] && !found; k++) found = excl_gids[k] == a;
            if (!found) return fail(NBX_EINVAL, "exclusion CSR is not symmetric");
        }
    ctx->natoms_global = n;
    ctx->ntypes = ntypes;
    const int nn = n > 0 ? n : 1;
    ctx->q_g.ensure(nn);
    ctx->type_g.ensure(nn);
    ctx->excl_off_g.ensure(n + 1);
    ctx->excl_gid_g.ensure(nexcl > 0 ? nexcl : 1);
    NBX_CUDA(cudaMemcpy(ctx->q_g.p, q, sizeof(float) * n, cudaMemcpyHostToDevice));
    NBX_CUDA(cudaMemcpy(ctx->type_g.p, type, sizeof(int) * n, cudaMemcpyHostToDevice));
    NBX_CUDA(cudaMemcpy(ctx->excl_off_g.p, excl_offsets, sizeof(int) * (n + 1), cudaMemcpyHostToDevice));
    if (nexcl > 0)
        NBX_CUDA(cudaMemcpy(ctx->excl_gid_g.p, excl_gids, sizeof(int) * nexcl, cudaMemcpyHostToDevice));
    std::vector<float2> t((size_t)ntypes * ntypes);
    const int lj = ctx->p.lj_modifier;
    if (lj == NBX_LJ_COMB_GEOM || lj == NBX_LJ_COMB_LB) {
        // combination rule: per-type parameters (nbx.h) replace the type-pair table
        t.resize(ntypes);
        for (int a = 0; a < ntypes; a++) {
            const double c6 = c6c12[2 * (a * ntypes + a)], c12 = c6c12[2 * (a * ntypes + a) + 1];
            if (c6 < 0.0 || c12 < 0.0) return fail(NBX_EINVAL, "negative LJ parameters");
            if (lj == NBX_LJ_COMB_GEOM) {
                t[a] = make_float2((float)std::sqrt(6.0 * c6), (float)std::sqrt(12.0 * c12));
            } else if (c6 > 0.0 && c12 > 0.0) {
                const double sig = std::sqrt(std::cbrt(c12 / c6)), eps = c6 * c6 / (4.0 * c12);
                t[a] = make_float2((float)(0.5 * sig), (float)std::sqrt(24.0 * eps));
            } else {
                if (c6 != 0.0 || c12 != 0.0)
                    return fail(NBX_EINVAL, "Lorentz-Berthelot needs c6 and c12 both zero or both positive");
                t[a] = make_float2(0.0f, 0.0f);
            }
        }
        for (int a = 0; a < ntypes; a++)
            for (int b = 0; b < ntypes; b++) {
                float p6, p12;
                if (lj == NBX_LJ_COMB_GEOM) {
                    p6 = t[a].x * t[b].x;
                    p12 = t[a].y * t[b].y;
                } else {
                    const float sg = t[a].x + t[b].x, s2 = sg * sg, s6 = (s2 * s2) * s2;
                    p6 = (t[a].y * t[b].y) * s6;
                    p12 = 2.0f * (p6 * s6);
                }
                const double w6 = 6.0 * c6c12[2 * (a * ntypes + b)], w12 = 12.0 * c6c12[2 * (a * ntypes + b) + 1];
                if (std::fabs(p6 - w6) > 1e-4 * std::fabs(w6) + 1e-30 || std::fabs(p12 - w12) > 1e-4 * std::fabs(w12) + 1e-30)
                    return fail(NBX_EINVAL, "LJ table does not follow the selected combination rule");
            }
    } else {
        for (int k = 0; k < ntypes * ntypes; k++)
            t[k] = make_float2(6.0f * c6c12[2 * k], 12.0f * c6c12[2 * k + 1]);
    }
    ctx->c6c12s.ensure(t.size());
    NBX_CUDA(cudaMemcpy(ctx->c6c12s.p, t.data(), sizeof(float2) * t.size(), cudaMemcpyHostToDevice));
    ctx->have_topology = true;
    ctx->epoch++;
    if (ctx->have_box)
        ctx->density = (double)n / ((double)ctx->box[0] * (double)ctx->box[1] * (double)ctx->box[2]);
    return NBX_OK;
    NBX_GUARD_END
}

NBX_API int nbx_set_box(nbx_ctx* ctx, const float box[3], const int32_t pbc[3])
{
    NBX_GUARD_BEGIN
    NBX_CHECK_CTX(ctx);
    if (!box) return fail(NBX_EINVAL, "null box");
    const float rmin = 2.0f * ctx->p.rlist_outer;
    for (int d = 0; d < 3; d++) {
        if (!(box[d] > 0.0f)) return fail(NBX_EINVAL, "box edges must be positive");
        const int per = pbc ? pbc[d] : 1;
        if (per && box[d] < rmin)
            return fail(NBX_EINVAL, "periodic box edge shorter than 2 * rlist_outer");
        ctx->box[d] = box[d];
        ctx->pbc[d] = per ? 1 : 0;
    }
    ctx->have_box = true;
    ctx->epoch++;
    if (ctx->have_topology)
        ctx->density = (double)ctx->natoms_global / ((double)box[0] * (double)box[1] * (double)box[2]);
    return NBX_OK;
    NBX_GUARD_END
}

NBX_API int nbx_grid_build(nbx_ctx* ctx, int grid, int32_t n, const float* x, const int32_t* gid,
                           const float lo[3], const float size[3], void* stream)
{
    NBX_GUARD_BEGIN
    NBX_CHECK_CTX(ctx);
    if (grid < 0 || grid > 1) return fail(NBX_EINVAL, "grid must be 0 or 1");
    if (!ctx->have_topology || !ctx->have_box) return fail(NBX_EINVAL, "set topology and box first");
    if (n < 0 || (n > 0 && !x) || !lo || !size) return fail(NBX_EINVAL, "bad grid arguments");
    if (grid == 0 && gid == nullptr && n != ctx->natoms_global)
        return fail(NBX_EINVAL, "identity gid requires n == natoms_global");
    for (int d = 0; d < 3; d++)
        if (!(size[d] > 0.0f)) return fail(NBX_EINVAL, "grid region size must be positive");
    grid_build(ctx, grid, n, x, gid, lo, size, (cudaStream_t)stream);
    ctx->epoch++;
    // a new grid invalidates the lists built on it
    ctx->list[0].built = ctx->list[0].built && grid != 0;
    ctx->list[1].built = false;
    return NBX_OK;
    NBX_GUARD_END
}

NBX_API int nbx_search(nbx_ctx* ctx, int list, void* stream)
{
    NBX_GUARD_BEGIN
    NBX_CHECK_CTX(ctx);
    if (list < 0 || list > 1) return fail(NBX_EINVAL, "list must be 0 or 1");
    if (!ctx->grid[0].built || (list == 1 && !ctx->grid[1].built))
        return fail(NBX_EINVAL, "build the grid(s) first");
    search(ctx, list, (cudaStream_t)stream);
    ctx->epoch++;
    return NBX_OK;
    NBX_GUARD_END
}

NBX_API int nbx_grid_search_pair(nbx_ctx* ctx, int32_t n_home, const float* x_home, const int32_t* gid_home,
                                 const float lo_home[3], const float size_home[3], int32_t n_halo,
                                 const float* x_halo, const int32_t* gid_halo, const float lo_halo[3],
                                 const float size_halo[3], void* stream, void* side_stream)
{
    NBX_GUARD_BEGIN
    NBX_CHECK_CTX(ctx);
    if (!ctx->have_topology || !ctx->have_box) return fail(NBX_EINVAL, "set topology and box first");
    if (n_home < 0 || n_halo < 0 || (n_home > 0 && !x_home) || (n_halo > 0 && !x_halo) || !lo_home ||
        !size_home || !lo_halo || !size_halo)
        return fail(NBX_EINVAL, "bad grid arguments");
    if (gid_home == nullptr && n_home != ctx->natoms_global)
        return fail(NBX_EINVAL, "identity gid requires n == natoms_global");
    for (int d = 0; d < 3; d++)
        if (!(size_home[d] > 0.0f) || !(size_halo[d] > 0.0f))
            return fail(NBX_EINVAL, "grid region size must be positive");
    cudaStream_t st0 = (cudaStream_t)stream, st1 = (cudaStream_t)side_stream;
    if (st0 == st1) return fail(NBX_EINVAL, "side_stream must differ from stream");
    if (!ctx->ev_pair[0]) {
        NBX_CUDA(cudaEventCreateWithFlags(&ctx->ev_pair[0], cudaEventDisableTiming));
        NBX_CUDA(cudaEventCreateWithFlags(&ctx->ev_pair[1], cudaEventDisableTiming));
    }
    ctx->list[0].built = false;
    ctx->list[1].built = false;
    // the inputs were produced in `stream` order: the side stream starts after them
    NBX_CUDA(cudaEventRecord(ctx->ev_pair[0], st0));
    NBX_CUDA(cudaStreamWaitEvent(st1, ctx->ev_pair[0], 0));
    const GridReq r[2] = {{n_home, x_home, gid_home, lo_home, size_home},
                          {n_halo, x_halo, gid_halo, lo_halo, size_halo}};
    grid_build_pair(ctx, r, st0, st1);
    ctx->epoch++;
    // the nonlocal list's i grid is grid 0
    NBX_CUDA(cudaEventRecord(ctx->ev_pair[0], st0));
    NBX_CUDA(cudaStreamWaitEvent(st1, ctx->ev_pair[0], 0));
    search_pair(ctx, st0, st1);
    NBX_CUDA(cudaEventRecord(ctx->ev_pair[1], st1));
    NBX_CUDA(cudaStreamWaitEvent(st0, ctx->ev_pair[1], 0));
    ctx->epoch++;
    return NBX_OK;
    NBX_GUARD_END
}

NBX_API int nbx_put_x(nbx_ctx* ctx, int grid, const float* x, void* stream)
{
    NBX_GUARD_BEGIN
    NBX_CHECK_CTX(ctx);
    if (grid < 0 || grid > 1 || !ctx->grid[grid].built) return fail(NBX_EINVAL, "grid not built");
    if (!x && ctx->grid[grid].n > 0) return fail(NBX_EINVAL, "null coordinates");
    put_x(ctx, grid, x, (cudaStream_t)stream);
    return NBX_OK;
    NBX_GUARD_END
}

NBX_API int nbx_prune(nbx_ctx* ctx, int list, int part, int nparts, void* stream)
{
    NBX_GUARD_BEGIN
    NBX_CHECK_CTX(ctx);
    if (list < 0 || list > 1 || !ctx->list[list].built) return fail(NBX_EINVAL, "list not built");
    if (nparts < 1 || part < 0 || part >= nparts) return fail(NBX_EINVAL, "bad prune part");
    prune(ctx, list, part, nparts, (cudaStream_t)stream);
    return NBX_OK;
    NBX_GUARD_END
}

NBX_API int nbx_force(nbx_ctx* ctx, int list, uint32_t flags, void* stream)
{
    NBX_GUARD_BEGIN
    NBX_CHECK_CTX(ctx);
    if (list < 0 || list > 1 || !ctx->list[list].built) return fail(NBX_EINVAL, "list not built");
    force(ctx, list, flags, (cudaStream_t)stream);
    return NBX_OK;
    NBX_GUARD_END
}

NBX_API int nbx_get_f(nbx_ctx* ctx, int grid, float* f, int accumulate, void* stream)
{
    NBX_GUARD_BEGIN
    NBX_CHECK_CTX(ctx);
    if (grid < 0 || grid > 1 || !ctx->grid[grid].built) return fail(NBX_EINVAL, "grid not built");
    if (!f && ctx->grid[grid].n > 0) return fail(NBX_EINVAL, "null force buffer");
    get_f(ctx, grid, f, accumulate, (cudaStream_t)stream);
    return NBX_OK;
    NBX_GUARD_END
}

// cached step graphs per context and kind (a caller that allocates fresh x / f tensors every
// step would otherwise grow the cache without bound)
static constexpr size_t kMaxStepGraphs = 16;

// X op (+ prune) + force + F op of a non-search MD step of the LOCAL list as one graph
// launch.  Captured (relaxed mode, on a private stream: nothing executes during capture)
// on first use for (x, f, what) and refreshed in place after anything bumped ctx->epoch.
NBX_API int nbx_step_graph(nbx_ctx* ctx, const float* x, float* f, uint32_t what, void* stream)
{
    NBX_GUARD_BEGIN
    NBX_CHECK_CTX(ctx);
    if (!ctx->list[0].built) return fail(NBX_EINVAL, "list not built");
    if (!x || !f) return fail(NBX_EINVAL, "null coordinates or force buffer");
    if (what & ~(uint32_t)NBX_STEP_PRUNE) return fail(NBX_EINVAL, "unknown step flags");
    nbx_ctx::StepGraph* g = nullptr;
    for (auto& e : ctx->graphs)
        if (e.x == x && e.f == f && e.what == what) g = &e;
    if (!g || g->epoch != ctx->epoch) {
        if (!ctx->cap_stream)
            NBX_CUDA(cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking));
        cudaStream_t cs = ctx->cap_stream;
        const int64_t l0 = ctx->launches;
        cudaGraph_t graph = nullptr;
        NBX_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed));
        try {
            put_x(ctx, 0, x, cs);
            if (what & NBX_STEP_PRUNE) prune(ctx, 0, 0, 1, cs);
            force(ctx, 0, 0, cs);
            get_f(ctx, 0, f, 0, cs);
        } catch (...) {
            cudaStreamEndCapture(cs, &graph);
            if (graph) cudaGraphDestroy(graph);
            ctx->launches = l0;
            throw;
        }
        NBX_CUDA(cudaStreamEndCapture(cs, &graph));
        const int kernels = (int)(ctx->launches - l0);
        ctx->launches = l0;
        bool updated = false;
        if (g) {
            cudaGraphExecUpdateResultInfo info;
            updated = cudaGraphExecUpdate(g->exec, graph, &info) == cudaSuccess;
            if (!updated) {
                cudaGetLastError();
                cudaGraphExecDestroy(g->exec);
            }
        } else {
            if (ctx->graphs.size() >= kMaxStepGraphs) { // callers cycling buffers: drop the oldest
                cudaGraphExecDestroy(ctx->graphs.front().exec);
                ctx->graphs.erase(ctx->graphs.begin());
            }
            ctx->graphs.push_back(nbx_ctx::StepGraph{x, f, what, 0, 0, nullptr});
            g = &ctx->graphs.back();
        }
        if (!updated) {
            cudaError_t e = cudaGraphInstantiate(&g->exec, graph, 0);
            if (e != cudaSuccess) {
                cudaGraphDestroy(graph);
                ctx->graphs.erase(ctx->graphs.begin() + (g - ctx->graphs.data()));
                NBX_CUDA(e);
            }
        }
        cudaGraphDestroy(graph);
        g->epoch = ctx->epoch;
        g->kernels = kernels;
    }
    NBX_CUDA(cudaGraphLaunch(g->exec, (cudaStream_t)stream));
    ctx->launches += g->kernels;
    return NBX_OK;
    NBX_GUARD_END
}

// One full GPU-resident non-search step as one graph launch: X op (+ prune) + force + PME on
// grid 0 (forces into the cluster buffer) + F op + leap-frog update of x and v in place.
// Captured like nbx_step_graph; refreshed after a search, a topology/box change or a PME box
// change.  For small boxes, where the ~12 separate launches of the step dominate.
NBX_API int nbx_step_graph_pme(nbx_ctx* ctx, nbx_pme* pme, float* x, float* f, float* v, const float* inv_mass,
                               float dt, uint32_t what, void* stream)
{
    NBX_GUARD_BEGIN
    NBX_CHECK_CTX(ctx);
    if (!pme || pme->device != ctx->device) return fail(NBX_EINVAL, "PME context missing or on another device");
    if (!pme->have_box) return fail(NBX_EINVAL, "PME box not set");
    if (!ctx->list[0].built) return fail(NBX_EINVAL, "list not built");
    if (!x || !f || !v || !inv_mass) return fail(NBX_EINVAL, "null buffer");
    if (what & ~(uint32_t)NBX_STEP_PRUNE) return fail(NBX_EINVAL, "unknown step flags");
    nbx_ctx::FullGraph* g = nullptr;
    for (auto& e : ctx->full_graphs)
        if (e.pme == pme && e.x == x && e.f == f && e.v == v && e.inv_mass == inv_mass && e.dt == dt &&
            e.what == what)
            g = &e;
    if (!g || g->epoch != ctx->epoch || g->pme_epoch != pme->epoch) {
        if (!ctx->cap_stream)
            NBX_CUDA(cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking));
        cudaStream_t cs = ctx->cap_stream;
        const int64_t l0 = ctx->launches, p0 = pme->launches;
        const int n = ctx->grid[0].n;
        cudaGraph_t graph = nullptr;
        NBX_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed));
        try {
            put_x(ctx, 0, x, cs);
            if (what & NBX_STEP_PRUNE) prune(ctx, 0, 0, 1, cs);
            force(ctx, 0, 0, cs);
            pme_compute_grid(pme, ctx, 0, 0u, cs);
            get_f(ctx, 0, f, 0, cs);
            leapfrog(n, x, v, f, inv_mass, dt, cs);
        } catch (...) {
            cudaStreamEndCapture(cs, &graph);
            if (graph) cudaGraphDestroy(graph);
            ctx->launches = l0;
            pme->launches = p0;
            throw;
        }
        NBX_CUDA(cudaStreamEndCapture(cs, &graph));
        const int kernels = (int)(ctx->launches - l0) + (int)(pme->launches - p0) + 1;
        ctx->launches = l0;
        pme->launches = p0;
        bool updated = false;
        if (g) {
            cudaGraphExecUpdateResultInfo info;
            updated = cudaGraphExecUpdate(g->exec, graph, &info) == cudaSuccess;
            if (!updated) {
                cudaGetLastError();
                cudaGraphExecDestroy(g->exec);
            }
        } else {
            if (ctx->full_graphs.size() >= kMaxStepGraphs) {
                cudaGraphExecDestroy(ctx->full_graphs.front().exec);
                ctx->full_graphs.erase(ctx->full_graphs.begin());
            }
            ctx->full_graphs.push_back(nbx_ctx::FullGraph{pme, 0, x, f, v, inv_mass, dt, what, 0, 0, nullptr});
            g = &ctx->full_graphs.back();
        }
        if (!updated) {
            cudaError_t e = cudaGraphInstantiate(&g->exec, graph, 0);
            if (e != cudaSuccess) {
                cudaGraphDestroy(graph);
                ctx->full_graphs.erase(ctx->full_graphs.begin() + (g - ctx->full_graphs.data()));
                NBX_CUDA(e);
            }
        }
        cudaGraphDestroy(graph);
        g->epoch = ctx->epoch;
        g->pme_epoch = pme->epoch;
        g->kernels = kernels;
    }
    NBX_CUDA(cudaGraphLaunch(g->exec, (cudaStream_t)stream));
    ctx->launches += g->kernels;
    return NBX_OK;
    NBX_GUARD_END
}

// ---- NVLink peer-memory halo (peer.cu) -------------------------------------------------
NBX_API int nbx_peer_init(nbx_ctx* ctx, int32_t rank, int32_t world, int32_t capacity, void* handle_out)
{
    NBX_GUARD_BEGIN
    NBX_CHECK_CTX(ctx);
    if (world < 1 || rank < 0 || rank >= world || capacity < 1 || !handle_out)
        return fail(NBX_EINVAL, "bad peer arguments");
    peer_init(ctx, rank, world, capacity, handle_out);
    return NBX_OK;
    NBX_GUARD_END
}

NBX_API int nbx_peer_open(nbx_ctx* ctx, const void* handles)
{
    NBX_GUARD_BEGIN
    NBX_CHECK_CTX(ctx);
    if (!handles) return fail(NBX_EINVAL, "null handles");
    peer_open(ctx, handles);
    return NBX_OK;
    NBX_GUARD_END
}

NBX_API int nbx_peer_set_halo(nbx_ctx* ctx, int32_t n_halo, const int32_t* owner, const int32_t* home,
                              const float* shift, void* stream)
{
    NBX_GUARD_BEGIN
    NBX_CHECK_CTX(ctx);
    if (n_halo < 0 || (n_halo > 0 && (!owner || !home || !shift))) return fail(NBX_EINVAL, "bad halo map");
    peer_set_halo(ctx, n_halo, owner, home, shift, (cudaStream_t)stream);
    ctx->epoch++;
    return NBX_OK;
    NBX_GUARD_END
}

NBX_API int nbx_peer_put_x(nbx_ctx* ctx, const float* x_home, uint32_t seq, void* stream)
{
    NBX_GUARD_BEGIN
    NBX_CHECK_CTX(ctx);
    if (!x_home && ctx->grid[0].n > 0) return fail(NBX_EINVAL, "null coordinates");
    peer_put_x(ctx, x_home, seq, (cudaStream_t)stream);
    return NBX_OK;
    NBX_GUARD_END
}

NBX_API int nbx_peer_halo_x(nbx_ctx* ctx, uint32_t seq, void* stream)
{
    NBX_GUARD_BEGIN
    NBX_CHECK_CTX(ctx);
    peer_halo_x(ctx, seq, (cudaStream_t)stream);
    return NBX_OK;
    NBX_GUARD_END
}

NBX_API int nbx_peer_force_nonlocal(nbx_ctx* ctx, uint32_t seq, uint32_t flags, void* stream)
{
    NBX_GUARD_BEGIN
    NBX_CHECK_CTX(ctx);
    if (flags & ~(uint32_t)(NBX_FORCE_ENERGY | NBX_FORCE_VIRIAL)) return fail(NBX_EINVAL, "bad force flags");
    peer_force_nonlocal(ctx, seq, flags, (cudaStream_t)stream);
    return NBX_OK;
    NBX_GUARD_END
}

NBX_API int nbx_peer_get_f(nbx_ctx* ctx, float* f_home, uint32_t seq, uint32_t flags, void* stream)
{
    NBX_GUARD_BEGIN
    NBX_CHECK_CTX(ctx);
    if (!f_home && ctx->grid[0].n > 0) return fail(NBX_EINVAL, "null force buffer");
    if (flags & ~(uint32_t)(NBX_FORCE_ENERGY | NBX_FORCE_VIRIAL)) return fail(NBX_EINVAL, "bad force flags");
    peer_get_f(ctx, f_home, seq, flags, (cudaStream_t)stream);
    return NBX_OK;
    NBX_GUARD_END
}

NBX_API int nbx_peer_status(nbx_ctx* ctx, int32_t* timed_out)
{
    NBX_GUARD_BEGIN
    NBX_CHECK_CTX(ctx);
    if (!timed_out) return fail(NBX_EINVAL, "null output");
    *timed_out = peer_status(ctx);
    return NBX_OK;
    NBX_GUARD_END
}

NBX_API int nbx_peer_repartition(nbx_ctx* ctx, const nbx_dd_geom* geom, const float* x_home, const int32_t* gid_home,
                                 int32_t n_home, uint32_t rseq, int32_t cap_ext, float* x_ext, int32_t* gid_ext,
                                 int32_t* owner, int32_t* home_index, float* shift, int32_t* n_home_out,
                                 int32_t* n_halo_out, void* stream)
{
    NBX_GUARD_BEGIN
    NBX_CHECK_CTX(ctx);
    if (!geom || !x_ext || !gid_ext || !owner || !home_index || !shift || !n_home_out || !n_halo_out ||
        n_home < 0 || (n_home > 0 && (!x_home || !gid_home)))
        return fail(NBX_EINVAL, "bad repartition arguments");
    if (peer_repartition(ctx, geom, x_home, gid_home, n_home, rseq, cap_ext, x_ext, gid_ext, owner, home_index, shift,
                         n_home_out, n_halo_out, (cudaStream_t)stream))
        return fail(NBX_ELIST_OVERFLOW, "repartition: new home / halo atoms exceed the capacities (counts returned)");
    ctx->epoch++;
    return NBX_OK;
    NBX_GUARD_END
}

NBX_API int nbx_clear_energies(nbx_ctx* ctx, void* stream)
{
    NBX_GUARD_BEGIN
    NBX_CHECK_CTX(ctx);
    NBX_CUDA(cudaMemsetAsync(ctx->acc.p, 0, sizeof(double) * (2 + 3 * NBX_NSHIFT + 9), (cudaStream_t)stream));
    ctx->xf_done = 0;
    return NBX_OK;
    NBX_GUARD_END
}

NBX_API int nbx_energies(nbx_ctx* ctx, double* e, double* vir, void* stream)
{
    NBX_GUARD_BEGIN
    NBX_CHECK_CTX(ctx);
    cudaStream_t st = (cudaStream_t)stream;
    const int NA = 2 + 3 * NBX_NSHIFT + 9;
    if (ctx->xf_done) {
        // peer-halo energy step: both grids' x (x) f were summed before their forces moved
        if (ctx->xf_done != 3u) return fail(NBX_EINVAL, "peer energy step incomplete (virial of one grid missing)");
    } else {
        NBX_CUDA(cudaMemsetAsync(ctx->acc.p + 2 + 3 * NBX_NSHIFT, 0, sizeof(double) * 9, st));
        virial_sum(ctx, 0, st);
        if (ctx->list[1].built) virial_sum(ctx, 1, st);
    }
    ctx->xf_done = 0;
    double h[2 + 3 * NBX_NSHIFT + 9];
    double q2 = 0.0;
    NBX_CUDA(cudaMemcpyAsync(h, ctx->acc.p, sizeof(double) * NA, cudaMemcpyDeviceToHost, st));
    NBX_CUDA(cudaMemcpyAsync(&q2, ctx->sumq2.p, sizeof(double), cudaMemcpyDeviceToHost, st));
    NBX_CUDA(cudaStreamSynchronize(st));
    double self;
    if (ctx->p.coulomb_type == NBX_COULOMB_EWALD || ctx->p.coulomb_type == NBX_COULOMB_EWALD_TAB)
        self = -(double)ctx->c.epsfac * q2 * (double)ctx->c.beta / std::sqrt(M_PI);
    else
        self = -0.5 * (double)ctx->c.epsfac * (double)ctx->c.c_rf * q2;
    if (e) {
        e[0] = h[0];
        e[1] = h[1] + self;
    }
    if (vir) {
        double w[9];
        for (int k = 0; k < 9; k++) w[k] = h[2 + 3 * NBX_NSHIFT + k];
        for (int s = 0; s < NBX_NSHIFT; s++) {
            const int sx = s % 3 - 1, sy = (s / 3) % 3 - 1, sz = s / 9 - 1;
            const float v[3] = {(float)sx * ctx->box[0], (float)sy * ctx->box[1], (float)sz * ctx->box[2]};
            for (int a = 0; a < 3; a++)
                for (int b = 0; b < 3; b++) w[3 * a + b] += (double)v[a] * h[2 + 3 * s + b];
        }
        for (int k = 0; k < 9; k++) vir[k] = -0.5 * w[k];
    }
    return NBX_OK;
    NBX_GUARD_END
}

NBX_API int nbx_grid_info_get(nbx_ctx* ctx, int grid, nbx_grid_info* out)
{
    if (!ctx || !out || grid < 0 || grid > 1) return fail(NBX_EINVAL, "bad arguments");
    const Grid& G = ctx->grid[grid];
    out->n = G.n;
    out->nslots = G.nslots;
    out->ncx = G.ncx;
    out->ncy = G.ncy;
    return NBX_OK;
}

NBX_API int nbx_grid_export(nbx_ctx* ctx, int grid, int32_t* order, float* xq, int32_t* type)
{
    NBX_GUARD_BEGIN
    NBX_CHECK_CTX(ctx);
    if (grid < 0 || grid > 1 || !ctx->grid[grid].built) return fail(NBX_EINVAL, "grid not built");
    Grid& G = ctx->grid[grid];
    NBX_CUDA(cudaDeviceSynchronize());
    if (order) NBX_CUDA(cudaMemcpy(order, G.order.p, sizeof(int) * G.nslots, cudaMemcpyDeviceToHost));
    if (xq) NBX_CUDA(cudaMemcpy(xq, G.xq.p, sizeof(float4) * G.nslots, cudaMemcpyDeviceToHost));
    if (type) NBX_CUDA(cudaMemcpy(type, G.type.p, sizeof(int) * G.nslots, cudaMemcpyDeviceToHost));
    return NBX_OK;
    NBX_GUARD_END
}

NBX_API int nbx_list_sizes_get(nbx_ctx* ctx, int list, nbx_list_sizes* out)
{
    NBX_GUARD_BEGIN
    NBX_CHECK_CTX(ctx);
    if (list < 0 || list > 1 || !out) return fail(NBX_EINVAL, "bad arguments");
    List& L = ctx->list[list];
    out->n_sci = L.built ? L.n_sci : 0;
    out->n_cj_outer = L.built ? L.n_cj : 0;
    out->n_pool = L.built ? L.n_pool : 0;
    out->n_cj_inner = 0;
    if (L.built && L.n_sci > 0) {
        NBX_CUDA(cudaDeviceSynchronize());
        std::vector<nbx_sci_entry> s(L.n_sci);
        NBX_CUDA(cudaMemcpy(s.data(), L.sci_in.p, sizeof(nbx_sci_entry) * L.n_sci, cudaMemcpyDeviceToHost));
        int64_t tot = 0;
        for (auto& e : s) tot += e.cj_end - e.cj_start;
        out->n_cj_inner = tot;
    }
    return NBX_OK;
    NBX_GUARD_END
}

NBX_API int nbx_list_export(nbx_ctx* ctx, int list, int which, nbx_sci_entry* sci, nbx_cj_entry* cj,
                            nbx_mask_pool_entry* pool)
{
    NBX_GUARD_BEGIN
    NBX_CHECK_CTX(ctx);
    if (list < 0 || list > 1 || !ctx->list[list].built) return fail(NBX_EINVAL, "list not built");
    List& L = ctx->list[list];
    NBX_CUDA(cudaDeviceSynchronize());
    if (pool) NBX_CUDA(cudaMemcpy(pool, L.pool.p, sizeof(nbx_mask_pool_entry) * L.n_pool, cudaMemcpyDeviceToHost));
    if (which == 0) {
        if (sci) NBX_CUDA(cudaMemcpy(sci, L.sci.p, sizeof(nbx_sci_entry) * L.n_sci, cudaMemcpyDeviceToHost));
        if (cj) NBX_CUDA(cudaMemcpy(cj, L.cj.p, sizeof(nbx_cj_entry) * L.n_cj, cudaMemcpyDeviceToHost));
        return NBX_OK;
    }
    std::vector<nbx_sci_entry> s(L.n_sci);
    std::vector<nbx_cj_entry> c(L.n_cj);
    if (L.n_sci) NBX_CUDA(cudaMemcpy(s.data(), L.sci_in.p, sizeof(nbx_sci_entry) * L.n_sci, cudaMemcpyDeviceToHost));
    if (L.n_cj) NBX_CUDA(cudaMemcpy(c.data(), L.cj_in.p, sizeof(nbx_cj_entry) * L.n_cj, cudaMemcpyDeviceToHost));
    int64_t pos = 0;
    for (int64_t e = 0; e < L.n_sci; e++) {
        nbx_sci_entry se = s[e];
        const int n = se.cj_end - se.cj_start;
        if (cj && n > 0) std::memcpy(cj + pos, c.data() + se.cj_start, sizeof(nbx_cj_entry) * n);
        if (sci) {
            sci[e] = se;
            sci[e].cj_start = (int32_t)pos;
            sci[e].cj_end = (int32_t)(pos + n);
        }
        pos += n;
    }
    return NBX_OK;
    NBX_GUARD_END
}

NBX_API int nbx_count_pairs(nbx_ctx* ctx, int list, int64_t* pairs, int64_t* slots, void* stream)
{
    NBX_GUARD_BEGIN
    NBX_CHECK_CTX(ctx);
    if (list < 0 || list > 1 || !ctx->list[list].built) return fail(NBX_EINVAL, "list not built");
    long long p = 0, s = 0;
    count_pairs(ctx, list, &p, &s, (cudaStream_t)stream);
    if (pairs) *pairs = p;
    if (slots) *slots = s;
    return NBX_OK;
    NBX_GUARD_END
}

NBX_API int nbx_fma_peak(nbx_ctx* ctx, double* tflops, void* stream)
{
    NBX_GUARD_BEGIN
    NBX_CHECK_CTX(ctx);
    if (!tflops) return fail(NBX_EINVAL, "null output");
    *tflops = fma_peak((cudaStream_t)stream);
    ctx->launches += 4;
    return NBX_OK;
    NBX_GUARD_END
}

NBX_API int64_t nbx_launch_count(nbx_ctx* ctx) { return ctx ? ctx->launches : -1; }

NBX_API int64_t nbx_alloc_count(void) { return (int64_t)__atomic_load_n(&g_allocs, __ATOMIC_RELAXED); }

NBX_API int nbx_halo_pack_x(const float* x, const int32_t* idx, int32_t n, const float shift[3],
                            float* out, void* stream)
{
    NBX_GUARD_BEGIN
    if (n < 0 || (n > 0 && (!x || !idx || !out || !shift))) return fail(NBX_EINVAL, "bad halo arguments");
    if (n == 0) return NBX_OK;
    halo_pack_x(x, idx, n, make_float3(shift[0], shift[1], shift[2]), out, (cudaStream_t)stream);
    return NBX_OK;
    NBX_GUARD_END
}

NBX_API int nbx_halo_unpack_add_f(float* f, const int32_t* idx, int32_t n, const float* in, void* stream)
{
    NBX_GUARD_BEGIN
    if (n < 0 || (n > 0 && (!f || !idx || !in))) return fail(NBX_EINVAL, "bad halo arguments");
    halo_unpack_add_f(f, idx, n, in, (cudaStream_t)stream);
    return NBX_OK;
    NBX_GUARD_END
}

// ---- row f4: PME and the leap-frog update (pme.cu) --------------------------------------
NBX_API int nbx_pme_create(int device, const nbx_pme_params* p, nbx_pme** out)
{
    NBX_GUARD_BEGIN
    if (!p || !out) return fail(NBX_EINVAL, "null argument");
    *out = nullptr;
    if (p->order != 4) return fail(NBX_EINVAL, "PME interpolation order must be 4");
    for (int d = 0; d < 3; d++)
        if (p->nk[d] < 8 || (p->nk[d] & 1)) return fail(NBX_EINVAL, "PME grid sizes must be even and >= 8");
    if (!(p->beta > 0.0f) || !(p->epsfac > 0.0f)) return fail(NBX_EINVAL, "PME beta and epsfac must be positive");
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev <= device || device < 0)
        return fail(NBX_ECUDA, std::string("no CUDA device ") + std::to_string(device) + " (" +
                                   cudaGetErrorString(e) + "); libnbx has no CPU fallback");
    cudaDeviceProp prop;
    NBX_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
        return fail(NBX_ECUDA, std::string("device ") + prop.name + " is not sm_100 (built for sm_100a only)");
    NBX_CUDA(cudaSetDevice(device));
    nbx_pme* pme = new nbx_pme();
    pme->device = device;
    for (int d = 0; d < 3; d++) pme->nk[d] = p->nk[d];
    pme->beta = p->beta;
    pme->epsfac = p->epsfac;
    try {
        pme_setup(pme);
    } catch (...) {
        pme_release(pme);
        delete pme;
        throw;
    }
    *out = pme;
    return NBX_OK;
    NBX_GUARD_END
}

NBX_API int nbx_pme_destroy(nbx_pme* pme)
{
    NBX_GUARD_BEGIN
    if (!pme) return NBX_OK;
    cudaSetDevice(pme->device);
    pme_release(pme);
    delete pme;
    return NBX_OK;
    NBX_GUARD_END
}

NBX_API int nbx_pme_set_box(nbx_pme* pme, const float box[3])
{
    NBX_GUARD_BEGIN
    NBX_CHECK_CTX(pme);
    if (!box) return fail(NBX_EINVAL, "null box");
    for (int d = 0; d < 3; d++)
        if (!(box[d] > 0.0f)) return fail(NBX_EINVAL, "box edges must be positive");
    pme_set_box(pme, box);
    return NBX_OK;
    NBX_GUARD_END
}

NBX_API int nbx_pme_compute(nbx_pme* pme, int32_t n, const float* x, const float* q, float* f, uint32_t flags,
                            void* stream)
{
    NBX_GUARD_BEGIN
    NBX_CHECK_CTX(pme);
    if (!pme->have_box) return fail(NBX_EINVAL, "PME compute before set_box");
    if (n < 0 || (n > 0 && (!x || !q || !f))) return fail(NBX_EINVAL, "bad PME arguments");
    pme_compute(pme, n, x, q, f, flags, (cudaStream_t)stream);
    return NBX_OK;
    NBX_GUARD_END
}

NBX_API int nbx_pme_compute_grid(nbx_pme* pme, nbx_ctx* ctx, int grid, uint32_t flags, void* stream)
{
    NBX_GUARD_BEGIN
    NBX_CHECK_CTX(pme);
    if (!ctx || ctx->device != pme->device) return fail(NBX_EINVAL, "PME and nonbonded contexts on different devices");
    if (grid < 0 || grid > 1) return fail(NBX_EINVAL, "bad grid index");
    if (!pme->have_box) return fail(NBX_EINVAL, "PME compute before set_box");
    pme_compute_grid(pme, ctx, grid, flags, (cudaStream_t)stream);
    return NBX_OK;
    NBX_GUARD_END
}

NBX_API int nbx_pme_energy(nbx_pme* pme, double* e_host, double* virial_host, void* stream)
{
    NBX_GUARD_BEGIN
    NBX_CHECK_CTX(pme);
    pme_energy(pme, e_host, virial_host, (cudaStream_t)stream);
    return NBX_OK;
    NBX_GUARD_END
}

NBX_API int64_t nbx_pme_launch_count(nbx_pme* pme) { return pme ? pme->launches : -1; }

NBX_API int nbx_pme_profile(nbx_pme* pme, int32_t n, const float* x, const float* q, float* f, float* ms_host,
                            void* stream)
{
    NBX_GUARD_BEGIN
    NBX_CHECK_CTX(pme);
    if (!pme->have_box) return fail(NBX_EINVAL, "PME profile before set_box");
    if (!ms_host || n < 0 || (n > 0 && (!x || !q || !f))) return fail(NBX_EINVAL, "bad PME arguments");
    pme_profile(pme, n, x, q, f, ms_host, (cudaStream_t)stream);
    return NBX_OK;
    NBX_GUARD_END
}

NBX_API int nbx_leapfrog(int32_t n, float* x, float* v, const float* f, const float* inv_mass, float dt, void* stream)
{
    NBX_GUARD_BEGIN
    if (n < 0 || (n > 0 && (!x || !v || !f || !inv_mass))) return fail(NBX_EINVAL, "bad leap-frog arguments");
    leapfrog(n, x, v, f, inv_mass, dt, (cudaStream_t)stream);
    return NBX_OK;
    NBX_GUARD_END
}

} // extern "C"
