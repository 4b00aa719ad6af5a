// bufops.cu -- X/F buffer ops, virial reduction, halo pack/unpack and the FFMA peak probe.
//
//  put_x   X buffer op (folded into NBNXM_* in the reference model, pipeline.py:231):
//          cluster-ordered xyzq from user-order x with the search-time wrap shifts.
//  get_f   F buffer op, KernelKind.REDUCE_FORCES (costs.py:41,172; pipeline.py:250-254,398-401):
//          cluster forces -> user order (gather by input atom), then the cluster buffer is cleared.
//  halo    KernelKind.HALO_PACK_UNPACK (costs.py:43,174; pipeline.py:366-379, 406-417).
// All of these are HBM/L2-bandwidth bound gathers/scatters: one thread per slot, float4
// accesses on the cluster side.
#include "nbx_internal.cuh"

namespace nbx {

__global__ void k_put_x(int nslots, const int* __restrict__ order, const float4* __restrict__ wrapk,
                        const float* __restrict__ x, float3 box, float4* __restrict__ xq)
{
    int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= nslots) return;
    int a = order[s];
    if (a < 0) return;
    float4 k = wrapk[s];
    float x0 = x[3 * a], x1 = x[3 * a + 1], x2 = x[3 * a + 2];
    xq[s] = make_float4(__fmaf_rn(-k.x, box.x, x0), __fmaf_rn(-k.y, box.y, x1),
                        __fmaf_rn(-k.z, box.z, x2), k.w);
}

// gather form: one thread per input atom, coalesced 12-byte writes of f, one 16-byte read of
// its cluster slot; the cluster buffer is cleared afterwards with a memset
__global__ void k_get_f(int n, const int* __restrict__ islot, const float4* __restrict__ fc,
                        float* __restrict__ f, int accumulate)
{
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= n) return;
    NBX_DCHECK(islot[a] >= 0);
    const float4 v = fc[islot[a]];
    if (accumulate) {
        f[3 * a] += v.x;
        f[3 * a + 1] += v.y;
        f[3 * a + 2] += v.z;
    } else {
        f[3 * a] = v.x;
        f[3 * a + 1] = v.y;
        f[3 * a + 2] = v.z;
    }
}

// sum over real slots of x (x) f in fp64 -> acc[0..8]
// sum over slots of (x - c) (x) f, c = the box centre: equal to sum x (x) f because the pair
// forces sum to zero (Newton III), but the fp32 force roundings' net sum no longer enters
// multiplied by the mean position (about half the error on a small box whose virial cancels
// to ~1e-3 of sum |x (x) f|)
__global__ void k_virial(int nslots, const int* __restrict__ order, const float4* __restrict__ xq,
                         const float4* __restrict__ fc, double3 c, double* acc)
{
    double w[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < nslots; s += gridDim.x * blockDim.x) {
        if (order[s] < 0) continue;
        float4 x = xq[s], f = fc[s];
        double xv[3] = {(double)x.x - c.x, (double)x.y - c.y, (double)x.z - c.z}, fv[3] = {f.x, f.y, f.z};
#pragma unroll
        for (int a = 0; a < 3; a++)
#pragma unroll
            for (int b = 0; b < 3; b++) w[3 * a + b] += xv[a] * fv[b];
    }
    __shared__ double sw[9];
    if (threadIdx.x < 9) sw[threadIdx.x] = 0.0;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 9; k++) {
        double v = w[k];
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if ((threadIdx.x & 31) == 0) atomicAdd(&sw[k], v);
    }
    __syncthreads();
    if (threadIdx.x < 9) atomicAdd(&acc[threadIdx.x], sw[threadIdx.x]);
}

__global__ void k_halo_pack(const float* __restrict__ x, const int* __restrict__ idx, int n,
                            float3 sh, float* __restrict__ out)
{
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    int a = idx[k];
    out[3 * k] = x[3 * a] + sh.x;
    out[3 * k + 1] = x[3 * a + 1] + sh.y;
    out[3 * k + 2] = x[3 * a + 2] + sh.z;
}

__global__ void k_halo_unpack_add(float* __restrict__ f, const int* __restrict__ idx, int n,
                                  const float* __restrict__ in)
{
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    int a = idx[k];
    f[3 * a] += in[3 * k];
    f[3 * a + 1] += in[3 * k + 1];
    f[3 * a + 2] += in[3 * k + 2];
}

void put_x(nbx_ctx* ctx, int g, const float* x, cudaStream_t st)
{
    Grid& G = ctx->grid[g];
    if (!G.built) throw CudaError{cudaErrorInvalidValue, "put_x before grid build"};
    if (G.nslots == 0) return;
    k_put_x<<<(G.nslots + 255) / 256, 256, 0, st>>>(G.nslots, G.order.p, G.wrapk.p, x,
                                                   make_float3(ctx->box[0], ctx->box[1], ctx->box[2]),
                                                   G.xq.p);
    ctx->launches++;
    NBX_CUDA(cudaGetLastError());
}

void get_f(nbx_ctx* ctx, int g, float* f, int accumulate, cudaStream_t st)
{
    Grid& G = ctx->grid[g];
    if (!G.built) throw CudaError{cudaErrorInvalidValue, "get_f before grid build"};
    if (G.nslots == 0) return;
    if (G.n > 0) {
        k_get_f<<<(G.n + 255) / 256, 256, 0, st>>>(G.n, G.islot.p, G.f.p, f, accumulate);
        ctx->launches++;
        NBX_CUDA(cudaGetLastError());
    }
    NBX_CUDA(cudaMemsetAsync(G.f.p, 0, sizeof(float4) * G.nslots, st));
}

void virial_sum(nbx_ctx* ctx, int g, cudaStream_t st)
{
    Grid& G = ctx->grid[g];
    if (!G.built || G.nslots == 0) return;
    int blocks = (G.nslots + 255) / 256;
    if (blocks > 4 * ctx->num_sms) blocks = 4 * ctx->num_sms;
    const double3 c = make_double3(0.5 * ctx->box[0], 0.5 * ctx->box[1], 0.5 * ctx->box[2]);
    k_virial<<<blocks, 256, 0, st>>>(G.nslots, G.order.p, G.xq.p, G.f.p, c, ctx->acc.p + 2 + 3 * NBX_NSHIFT);
    ctx->launches++;
    NBX_CUDA(cudaGetLastError());
}

void halo_pack_x(const float* x, const int* idx, int n, float3 shift, float* out, cudaStream_t st)
{
    if (n <= 0) return;
    k_halo_pack<<<(n + 255) / 256, 256, 0, st>>>(x, idx, n, shift, out);
    NBX_CUDA(cudaGetLastError());
}

void halo_unpack_add_f(float* f, const int* idx, int n, const float* in, cudaStream_t st)
{
    if (n <= 0) return;
    k_halo_unpack_add<<<(n + 255) / 256, 256, 0, st>>>(f, idx, n, in);
    NBX_CUDA(cudaGetLastError());
}

// ---- FP32 FFMA peak probe (roofline denominator) ------------------
__global__ void k_ffma_peak(float* out, float a, float b, int iters)
{
    float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5,
          x6 = x0 + 6, x7 = x0 + 7;
    const float y0 = a * x0, y1 = b * x1;
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int k = 0; k < 16; k++) {
            x0 = fmaf(x0, y0, y1); x1 = fmaf(x1, y1, y0); x2 = fmaf(x2, y0, y1); x3 = fmaf(x3, y1, y0);
            x4 = fmaf(x4, y0, y1); x5 = fmaf(x5, y1, y0); x6 = fmaf(x6, y0, y1); x7 = fmaf(x7, y1, y0);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

double fma_peak(cudaStream_t st)
{
    int dev = 0, sms = 0;
    NBX_CUDA(cudaGetDevice(&dev));
    NBX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int blocks = sms * 8, threads = 256, iters = 2000;
    float* out = nullptr;
    NBX_CUDA(cudaMalloc(&out, sizeof(float) * blocks * threads));
    cudaEvent_t e0, e1;
    NBX_CUDA(cudaEventCreate(&e0));
    NBX_CUDA(cudaEventCreate(&e1));
    double best = 0.0;
    for (int rep = 0; rep < 4; rep++) {
        NBX_CUDA(cudaEventRecord(e0, st));
        k_ffma_peak<<<blocks, threads, 0, st>>>(out, 1.0001f, 0.9999f, iters);
        NBX_CUDA(cudaEventRecord(e1, st));
        NBX_CUDA(cudaEventSynchronize(e1));
        float ms = 0.f;
        NBX_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        double fl = 2.0 * blocks * threads * (double)iters * 16 * 8;
        double tf = fl / (ms * 1e-3) / 1e12;
        if (rep > 0 && tf > best) best = tf;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    return best;
}

} // namespace nbx
