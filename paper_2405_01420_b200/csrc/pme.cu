// pme.cu -- smooth particle-mesh Ewald (row f4) and the leap-frog update on sm_100a.
//
// The reciprocal-space half of the Ewald electrostatics, as the reference submits it after the
// nonbonded kernels (pipeline.py:241-246): PME_SPREAD -> FFT_3D_FORWARD -> PME_SOLVE ->
// FFT_3D_INVERSE -> PME_GATHER, with GRID_MEMSET (pipeline.py:256-257) and LEAP_FROG
// (pipeline.py:249-251).  Algorithm and conventions: oracle/pme.py (its docstring is the spec).
//
// sm_100a design:
//  * spread / gather: 4 threads per atom (one z spline point each, the 16 (x, y) points in a
//    loop), so 4 adjacent threads touch 4 consecutive z points; charges are added with
//    red.global.add.f32 into the grid (the 12M-atom grid, 420^3 fp32 = 296 MB, streams
//    through L2 in the input's spatial order); gather reduces the 4 partial forces with 2 xor
//    shuffles (16 threads per atom, measured first, spent most of their time recomputing the
//    B-spline weights: spread 1.50 / gather 2.11 ms on 12 M atoms);
//  * the B-spline weights are recomputed in each kernel instead of stored: 96 bytes per atom
//    of HBM traffic saved twice;
//  * FFTs: cuFFT single-precision R2C / C2R plans, unnormalised, out of place (library call,
//    like cuBLAS for a plain GEMM);
//  * solve: one thread per half-spectrum element on a 3-D launch grid, influence function from
//    per-dimension modulus and Gaussian tables, fp64 block reduction of the energy and virial
//    (energy steps only);
//  * no CPU fallback: the context refuses to exist without an sm_100 device (capi.cu).
#include <atomic>
#include <cmath>
#include <vector>

#include "nbx_internal.cuh"

namespace nbx {

constexpr int PME_THREADS = 256; // 16 atoms per block in spread / gather

struct PmeGeom {
    int nx, ny, nz;
    float bx, by, bz;    // box
    float ibx, iby, ibz; // 1 / box
};

// B-spline weights theta_j = M_4(w + j) and derivatives M_3(w + j) - M_3(w + j - 1), j = 0..3
// (oracle/pme.py splines(): the recursion in closed form for order 4)
__device__ __forceinline__ void bspline4(float w, float th[4], float dth[4])
{
    const float w2 = w * w, w3 = w2 * w, v = 1.0f - w;
    th[0] = w3 * (1.0f / 6.0f);
    th[1] = (-3.0f * w3 + 3.0f * w2 + 3.0f * w + 1.0f) * (1.0f / 6.0f);
    th[2] = (3.0f * w3 - 6.0f * w2 + 4.0f) * (1.0f / 6.0f);
    th[3] = v * v * v * (1.0f / 6.0f);
    dth[0] = 0.5f * w2;
    dth[1] = (-3.0f * w2 + 2.0f * w + 1.0f) * 0.5f;
    dth[2] = (3.0f * w2 - 4.0f * w) * 0.5f;
    dth[3] = -0.5f * v * v;
}

// u = K frac(x / L); base = floor(u) (clamped to K-1), w = u - base
__device__ __forceinline__ void frac_index(float x, float ib, int K, int& base, float& w)
{
    float f = x * ib;
    f -= floorf(f);
    const float u = f * (float)K;
    int b = (int)u;
    b = min(b, K - 1);
    base = b;
    w = u - (float)b;
}

__device__ __forceinline__ int wrapk(int i, int K) { return i < 0 ? i + K : i; }

// element j of a 4-vector held in registers (selects, no local-memory indexing)
__device__ __forceinline__ float sel4(const float v[4], int j)
{
    return j == 0 ? v[0] : (j == 1 ? v[1] : (j == 2 ? v[2] : v[3]));
}

// atom a's position and charge: [n][3] + [n] arrays, or (XQ4) the nonbonded grid's
// cluster-ordered float4 (x, y, z, q) buffer (fillers have q = 0 and are skipped)
template <bool XQ4>
__device__ __forceinline__ void load_atom(int a, const float* __restrict__ x, const float* __restrict__ q, float& px,
                                          float& py, float& pz, float& qa)
{
    if (XQ4) {
        const float4 t = reinterpret_cast<const float4*>(x)[a];
        px = t.x;
        py = t.y;
        pz = t.z;
        qa = t.w;
    } else {
        px = x[3 * a + 0];
        py = x[3 * a + 1];
        pz = x[3 * a + 2];
        qa = q[a];
    }
}

// 4 threads per atom (one z spline point each, 16 (x, y) points in a loop): 4 adjacent threads
// add into 4 consecutive z points, and the B-spline weights are computed 4x per atom, not 16x
template <bool XQ4>
__global__ void __launch_bounds__(PME_THREADS) k_pme_spread(int n, const float* __restrict__ x,
                                                            const float* __restrict__ q, PmeGeom g,
                                                            float* __restrict__ grid)
{
    const int a = (blockIdx.x * PME_THREADS + threadIdx.x) >> 2;
    const int jz = threadIdx.x & 3;
    if (a >= n) return;
    float px, py, pz, qa;
    load_atom<XQ4>(a, x, q, px, py, pz, qa);
    if (qa == 0.0f) return;
    int ix, iy, iz;
    float wx, wy, wz, tx[4], ty[4], tz[4], d[4];
    frac_index(px, g.ibx, g.nx, ix, wx);
    frac_index(py, g.iby, g.ny, iy, wy);
    frac_index(pz, g.ibz, g.nz, iz, wz);
    bspline4(wx, tx, d);
    bspline4(wy, ty, d);
    bspline4(wz, tz, d);
    const float qz = qa * sel4(tz, jz);
    float* col = grid + wrapk(iz - jz, g.nz);
#pragma unroll
    for (int jx = 0; jx < 4; jx++) {
        float* plane = col + (size_t)wrapk(ix - jx, g.nx) * g.ny * g.nz;
        const float qxz = qz * tx[jx];
#pragma unroll
        for (int jy = 0; jy < 4; jy++) atomicAdd(plane + (size_t)wrapk(iy - jy, g.ny) * g.nz, qxz * ty[jy]);
    }
}

// one thread per half-spectrum element on a (z, y, x) launch grid (no index divisions); the
// Gaussian factor is a product of per-dimension tables: G = ex[x] ey[y] ez[z] / (pi V m^2) b
__global__ void __launch_bounds__(256) k_pme_solve(PmeGeom g, float beta, float epsfac, float2* __restrict__ spec,
                                                   const float* __restrict__ bmod, const float* __restrict__ gex,
                                                   int energy, double* acc)
{
    const int nzh = g.nz / 2 + 1;
    const int z = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y, xi = blockIdx.z;
    double ev[7] = {0, 0, 0, 0, 0, 0, 0}; // E, xx, yy, zz, xy, xz, yz
    if (z < nzh) {
        const long long e = ((long long)xi * g.ny + y) * nzh + z;
        const int mx = xi <= g.nx / 2 ? xi : xi - g.nx;
        const int my = y <= g.ny / 2 ? y : y - g.ny;
        const float tx = (float)mx * g.ibx, ty = (float)my * g.iby, tz = (float)z * g.ibz;
        const float m2 = tx * tx + ty * ty + tz * tz;
        const float pi = 3.14159265358979f;
        float G = 0.0f;
        if (e != 0) {
            const float b = bmod[xi] * bmod[g.nx + y] * bmod[g.nx + g.ny + z];
            const float ex = gex[xi] * gex[g.nx + y] * gex[g.nx + g.ny + z];
            G = __fdividef(ex * b, pi * (g.bx * g.by * g.bz) * m2);
        }
        float2 s = spec[e];
        if (energy && e != 0) {
            const float w = (z == 0 || (2 * z == g.nz)) ? 1.0f : 2.0f;
            const double em = 0.5 * (double)epsfac * (double)G * ((double)s.x * s.x + (double)s.y * s.y) * w;
            const double fac = 2.0 * (1.0 + (double)pi * pi * m2 / ((double)beta * beta)) / (double)m2;
            ev[0] = em;
            ev[1] = -0.5 * em * (1.0 - fac * tx * tx);
            ev[2] = -0.5 * em * (1.0 - fac * ty * ty);
            ev[3] = -0.5 * em * (1.0 - fac * tz * tz);
            ev[4] = 0.5 * em * fac * tx * ty;
            ev[5] = 0.5 * em * fac * tx * tz;
            ev[6] = 0.5 * em * fac * ty * tz;
        }
        s.x *= G;
        s.y *= G;
        spec[e] = s;
    }
    if (energy) {
        __shared__ double red[7][8];
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
        for (int k = 0; k < 7; k++) {
            double v = ev[k];
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0) red[k][w] = v;
        }
        __syncthreads();
        if (threadIdx.x < 7) {
            double v = 0.0;
            for (int k = 0; k < (int)(blockDim.x >> 5); k++) v += red[threadIdx.x][k];
            if (v != 0.0) atomicAdd(acc + threadIdx.x, v);
        }
    }
}

// 4 threads per atom (one z spline point each, 16 (x, y) points), 2 xor shuffles
// XQ4: forces are added to the nonbonded grid's cluster force buffer (float4 per slot), which
// the F buffer op then returns in the caller's atom order together with the nonbonded forces
template <bool XQ4>
__global__ void __launch_bounds__(PME_THREADS) k_pme_gather(int n, const float* __restrict__ x,
                                                            const float* __restrict__ q, PmeGeom g, float epsfac,
                                                            const float* __restrict__ phi, float* __restrict__ f)
{
    const int a = (blockIdx.x * PME_THREADS + threadIdx.x) >> 2;
    const int jz = threadIdx.x & 3;
    const bool live = a < n;
    const int ac = live ? a : n - 1;
    float px, py, pz, qa;
    load_atom<XQ4>(ac, x, q, px, py, pz, qa);
    int ix, iy, iz;
    float wx, wy, wz, tx[4], ty[4], tz[4], dx[4], dy[4], dz[4];
    frac_index(px, g.ibx, g.nx, ix, wx);
    frac_index(py, g.iby, g.ny, iy, wy);
    frac_index(pz, g.ibz, g.nz, iz, wz);
    bspline4(wx, tx, dx);
    bspline4(wy, ty, dy);
    bspline4(wz, tz, dz);
    const float tz1 = sel4(tz, jz), dz1 = sel4(dz, jz);
    const float* col = phi + wrapk(iz - jz, g.nz);
    float sx = 0.f, sy = 0.f, sz = 0.f;
#pragma unroll
    for (int jx = 0; jx < 4; jx++) {
        const float* plane = col + (size_t)wrapk(ix - jx, g.nx) * g.ny * g.nz;
        float px = 0.f, py = 0.f, pz = 0.f; // sums over y at fixed x
#pragma unroll
        for (int jy = 0; jy < 4; jy++) {
            const float p = __ldg(plane + (size_t)wrapk(iy - jy, g.ny) * g.nz);
            px = fmaf(ty[jy], p, px);
            py = fmaf(dy[jy], p, py);
        }
        pz = px;
        sx = fmaf(dx[jx], px, sx);
        sy = fmaf(tx[jx], py, sy);
        sz = fmaf(tx[jx], pz, sz);
    }
    sx *= tz1;
    sy *= tz1;
    sz *= dz1;
#pragma unroll
    for (int o = 2; o > 0; o >>= 1) {
        sx += __shfl_xor_sync(0xffffffffu, sx, o);
        sy += __shfl_xor_sync(0xffffffffu, sy, o);
        sz += __shfl_xor_sync(0xffffffffu, sz, o);
    }
    if (live && jz == 0 && qa != 0.0f) {
        const float s = -epsfac * qa;
        float* fa = f + (XQ4 ? 4 : 3) * a;
        fa[0] += s * (float)g.nx * g.ibx * sx;
        fa[1] += s * (float)g.ny * g.iby * sy;
        fa[2] += s * (float)g.nz * g.ibz * sz;
    }
}

__global__ void k_leapfrog(int n, float* __restrict__ x, float* __restrict__ v, const float* __restrict__ f,
                           const float* __restrict__ im, float dt)
{
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= 3 * n) return;
    const float vn = fmaf(f[k] * im[k / 3], dt, v[k]);
    v[k] = vn;
    x[k] = fmaf(vn, dt, x[k]);
}

// host-side modulus |b(m)|^2 (oracle/pme.py bsp_moduli), double, rounded once
static void bsp_moduli(int K, std::vector<float>& out, int count)
{
    const double mk[3] = {1.0 / 6.0, 4.0 / 6.0, 1.0 / 6.0}; // M_4(1), M_4(2), M_4(3)
    for (int m = 0; m < count; m++) {
        double re = 0.0, im = 0.0;
        for (int k = 0; k < 3; k++) {
            const double a = 2.0 * M_PI * m * k / K;
            re += mk[k] * std::cos(a);
            im += mk[k] * std::sin(a);
        }
        out.push_back((float)(1.0 / (re * re + im * im)));
    }
}

void pme_setup(nbx_pme* pme)
{
    const int nx = pme->nk[0], ny = pme->nk[1], nz = pme->nk[2];
    pme->grid.ensure((size_t)nx * ny * nz);
    pme->spec.ensure((size_t)nx * ny * (nz / 2 + 1));
    std::vector<float> b;
    bsp_moduli(nx, b, nx);
    bsp_moduli(ny, b, ny);
    bsp_moduli(nz, b, nz / 2 + 1);
    pme->bmod.ensure(b.size());
    NBX_CUDA(cudaMemcpy(pme->bmod.p, b.data(), sizeof(float) * b.size(), cudaMemcpyHostToDevice));
    pme->gex.ensure(b.size());
    pme->acc.ensure(10);
    NBX_CUDA(cudaMemset(pme->acc.p, 0, sizeof(double) * 10));
    if (cufftPlan3d(&pme->fwd, nx, ny, nz, CUFFT_R2C) != CUFFT_SUCCESS ||
        cufftPlan3d(&pme->inv, nx, ny, nz, CUFFT_C2R) != CUFFT_SUCCESS)
        throw CudaError{cudaErrorMemoryAllocation, "cufftPlan3d"};
}

void pme_set_box(nbx_pme* pme, const float box[3])
{
    for (int d = 0; d < 3; d++) pme->box[d] = box[d];
    pme->have_box = true;
    // process-wide counter: a PME context created later at a freed one's address never
    // matches a graph captured against the old one
    static std::atomic<uint64_t> box_epoch{1};
    pme->epoch = ++box_epoch;
    // per-dimension Gaussian factors exp(-pi^2 mt_d^2 / beta^2), mt_d = m_d / L_d (m_d signed)
    std::vector<float> t;
    const double pb = M_PI / (double)pme->beta;
    for (int d = 0; d < 3; d++) {
        const int K = pme->nk[d], cnt = d < 2 ? K : K / 2 + 1;
        for (int m = 0; m < cnt; m++) {
            const int ms = (d < 2 && m > K / 2) ? m - K : m;
            const double mt = (double)ms / (double)box[d];
            t.push_back((float)std::exp(-pb * pb * mt * mt));
        }
    }
    NBX_CUDA(cudaMemcpy(pme->gex.p, t.data(), sizeof(float) * t.size(), cudaMemcpyHostToDevice));
}

static PmeGeom geom(const nbx_pme* pme)
{
    PmeGeom g;
    g.nx = pme->nk[0];
    g.ny = pme->nk[1];
    g.nz = pme->nk[2];
    g.bx = pme->box[0];
    g.by = pme->box[1];
    g.bz = pme->box[2];
    g.ibx = 1.0f / g.bx;
    g.iby = 1.0f / g.by;
    g.ibz = 1.0f / g.bz;
    return g;
}

// ev (optional, 7 events): recorded before the memset and after each of the 6 stages
// (memset, spread, R2C, solve, C2R, gather) -- nbx_pme_profile's per-stage times
void pme_compute(nbx_pme* pme, int n, const float* x, const float* q, float* f, unsigned flags, cudaStream_t st,
                 cudaEvent_t* ev, bool xq4)
{
    const PmeGeom g = geom(pme);
    const size_t ng = (size_t)g.nx * g.ny * g.nz;
    if (ev) NBX_CUDA(cudaEventRecord(ev[0], st));
    NBX_CUDA(cudaMemsetAsync(pme->grid.p, 0, sizeof(float) * ng, st)); // GRID_MEMSET
    if (ev) NBX_CUDA(cudaEventRecord(ev[1], st));
    const int blocks = (int)(((long long)n * 4 + PME_THREADS - 1) / PME_THREADS);
    if (n > 0) {
        if (xq4) k_pme_spread<true><<<blocks, PME_THREADS, 0, st>>>(n, x, q, g, pme->grid.p);
        else k_pme_spread<false><<<blocks, PME_THREADS, 0, st>>>(n, x, q, g, pme->grid.p);
    }
    NBX_CUDA(cudaGetLastError());
    if (ev) NBX_CUDA(cudaEventRecord(ev[2], st));
    if (cufftSetStream(pme->fwd, st) != CUFFT_SUCCESS || cufftSetStream(pme->inv, st) != CUFFT_SUCCESS)
        throw CudaError{cudaErrorInvalidValue, "cufftSetStream"};
    if (cufftExecR2C(pme->fwd, pme->grid.p, reinterpret_cast<cufftComplex*>(pme->spec.p)) != CUFFT_SUCCESS)
        throw CudaError{cudaErrorLaunchFailure, "cufftExecR2C"};
    if (ev) NBX_CUDA(cudaEventRecord(ev[3], st));
    const int energy = (flags & (NBX_FORCE_ENERGY | NBX_FORCE_VIRIAL)) != 0;
    const int nzh = g.nz / 2 + 1;
    const dim3 sgrid((nzh + 127) / 128, g.ny, g.nx);
    k_pme_solve<<<sgrid, 128, 0, st>>>(g, pme->beta, pme->epsfac, pme->spec.p, pme->bmod.p, pme->gex.p, energy,
                                       pme->acc.p);
    NBX_CUDA(cudaGetLastError());
    if (ev) NBX_CUDA(cudaEventRecord(ev[4], st));
    if (cufftExecC2R(pme->inv, reinterpret_cast<cufftComplex*>(pme->spec.p), pme->grid.p) != CUFFT_SUCCESS)
        throw CudaError{cudaErrorLaunchFailure, "cufftExecC2R"};
    if (ev) NBX_CUDA(cudaEventRecord(ev[5], st));
    if (n > 0) {
        if (xq4) k_pme_gather<true><<<blocks, PME_THREADS, 0, st>>>(n, x, q, g, pme->epsfac, pme->grid.p, f);
        else k_pme_gather<false><<<blocks, PME_THREADS, 0, st>>>(n, x, q, g, pme->epsfac, pme->grid.p, f);
    }
    NBX_CUDA(cudaGetLastError());
    if (ev) NBX_CUDA(cudaEventRecord(ev[6], st));
    pme->launches += (n > 0 ? 3 : 1);
}

void pme_profile(nbx_pme* pme, int n, const float* x, const float* q, float* f, float ms[6], cudaStream_t st)
{
    cudaEvent_t ev[7];
    for (int k = 0; k < 7; k++) NBX_CUDA(cudaEventCreate(&ev[k]));
    pme_compute(pme, n, x, q, f, 0u, st, ev);
    NBX_CUDA(cudaEventSynchronize(ev[6]));
    for (int k = 0; k < 6; k++) NBX_CUDA(cudaEventElapsedTime(&ms[k], ev[k], ev[k + 1]));
    for (int k = 0; k < 7; k++) cudaEventDestroy(ev[k]);
}

// PME on the atoms of a nonbonded context's grid, in its cluster order (spatially sorted:
// neighbouring atoms touch neighbouring grid points), forces into its cluster force buffer
void pme_compute_grid(nbx_pme* pme, nbx_ctx* ctx, int g, unsigned flags, cudaStream_t st)
{
    Grid& G = ctx->grid[g];
    if (!G.built) throw CudaError{cudaErrorInvalidValue, "PME on a grid before grid build"};
    pme_compute(pme, G.nslots, reinterpret_cast<const float*>(G.xq.p), nullptr, reinterpret_cast<float*>(G.f.p),
                flags, st, nullptr, true);
}

void pme_energy(nbx_pme* pme, double* e, double* vir, cudaStream_t st)
{
    double h[10];
    NBX_CUDA(cudaMemcpyAsync(h, pme->acc.p, sizeof(h), cudaMemcpyDeviceToHost, st));
    NBX_CUDA(cudaMemsetAsync(pme->acc.p, 0, sizeof(h), st));
    NBX_CUDA(cudaStreamSynchronize(st));
    if (e) *e = h[0];
    if (vir) {
        // acc: xx, yy, zz, xy, xz, yz -> row-major symmetric 3x3
        const double xx = h[1], yy = h[2], zz = h[3], xy = h[4], xz = h[5], yz = h[6];
        const double m[9] = {xx, xy, xz, xy, yy, yz, xz, yz, zz};
        for (int k = 0; k < 9; k++) vir[k] = m[k];
    }
}

void pme_release(nbx_pme* pme)
{
    if (pme->fwd) cufftDestroy(pme->fwd);
    if (pme->inv) cufftDestroy(pme->inv);
    pme->fwd = pme->inv = 0;
    pme->grid.release();
    pme->spec.release();
    pme->bmod.release();
    pme->gex.release();
    pme->acc.release();
}

void leapfrog(int n, float* x, float* v, const float* f, const float* inv_mass, float dt, cudaStream_t st)
{
    if (n <= 0) return;
    k_leapfrog<<<(3 * n + 255) / 256, 256, 0, st>>>(n, x, v, f, inv_mass, dt);
    NBX_CUDA(cudaGetLastError());
}

} // namespace nbx
