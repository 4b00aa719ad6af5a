// grid.cu -- grid build (first half of KernelKind.PAIR_SEARCH, costs.py:32; pipeline.py:226-230).
//
// Atoms are wrapped into the box (periodic dims), binned into x-y columns, sorted by
// (column, z, input index) with a stable 64-bit radix sort, and every column is padded to a
// multiple of 32 slots.  Each 32-slot slab (one super-cluster) is sub-sorted y -> x -> z
// into 2 x 2 x (2 x 4): halves of 16, j-clusters of 8, i-clusters of 4.
// Every floating-point operation that decides a bin or a slot is the exact op sequence of the
// CPU oracle (oracle/nbx_oracle.c ora_grid_build), so the layout is bit-identical.
#include <algorithm>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "nbx_internal.cuh"

namespace nbx {

struct BinArgs {
    int n;
    const float* x;
    float3 box, invL, lo;
    int pbc[3];
    float inv_cell[2];
    int ncx, ncy;
};

// what grid_end needs from grid_begin
struct GridStage {
    BinArgs B;
    const int* gid = nullptr;
    int* h = nullptr; // pinned: [0] padded slot count
};

__device__ __forceinline__ float wrap_k(float x, float invL, int pbc)
{
    return pbc ? floorf(__fmul_rn(x, invL)) : 0.0f;
}

__device__ __forceinline__ int cell_index(float xw, float lo, float inv, int nc)
{
    float t = floorf(__fmul_rn(__fsub_rn(xw, lo), inv));
    if (!(t >= 0.0f)) return 0;
    if (t > (float)(nc - 1)) return nc - 1;
    return (int)t;
}

__device__ __forceinline__ float3 wrap_atom(const float* x, int a, const BinArgs& A, float3& k)
{
    float x0 = x[3 * a], x1 = x[3 * a + 1], x2 = x[3 * a + 2];
    k.x = wrap_k(x0, A.invL.x, A.pbc[0]);
    k.y = wrap_k(x1, A.invL.y, A.pbc[1]);
    k.z = wrap_k(x2, A.invL.z, A.pbc[2]);
    return make_float3(__fmaf_rn(-k.x, A.box.x, x0), __fmaf_rn(-k.y, A.box.y, x1),
                       __fmaf_rn(-k.z, A.box.z, x2));
}

__global__ void k_bin(BinArgs A, unsigned long long* key, int* val, int* col_count)
{
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    const bool real = a < A.n;
    int col = -1;
    if (real) {
        float3 k;
        float3 w = wrap_atom(A.x, a, A, k);
        int cx = cell_index(w.x, A.lo.x, A.inv_cell[0], A.ncx);
        int cy = cell_index(w.y, A.lo.y, A.inv_cell[1], A.ncy);
        col = cx * A.ncy + cy;
        key[a] = ((unsigned long long)(unsigned)col << 32) | ordkey(w.z);
        val[a] = a;
    }
    // warp-aggregated column counts: consecutive input atoms (molecules, lattice rows) mostly
    // share a column, so one atomic per distinct column per warp instead of one per atom
    const unsigned peers = __match_any_sync(0xffffffffu, col);
    if (real && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&col_count[col], __popc(peers));
}

__global__ void k_pad(const int* col_count, int ncol, int* padded)
{
    int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c > ncol) return;
    padded[c] = c < ncol ? ((col_count[c] + 31) / 32) * 32 : 0;
}

struct SlabArgs {
    BinArgs B;
    int nsci, ncol;
    const int* col_start;  // slot offsets [ncol+1]
    const int* col_astart; // sorted-atom offsets [ncol+1]
    const int* col_count;
    const int* sorted;     // input indices in (col, z, idx) order
    const int* gid_in;     // may be null
    const float* q_g;
    const int* type_g;
    int* order;
    int* gid;
    int* type;
    float4* xq;
    float4* wrapk;
    int* slotmap;
    int* islot;
    int natoms_global; // slotmap extent (checked builds)
};

// rank of this lane's key among the real lanes of the same group (ties impossible: idx)
__device__ __forceinline__ int group_rank(unsigned long long key, int group, bool real)
{
    int r = 0;
#pragma unroll 8
    for (int l = 0; l < 32; l++) {
        unsigned long long ok = __shfl_sync(0xffffffffu, key, l);
        int og = __shfl_sync(0xffffffffu, group, l);
        int oreal = __shfl_sync(0xffffffffu, (int)real, l);
        r += (oreal && og == group && ok < key) ? 1 : 0;
    }
    return r;
}

__global__ void k_slab(SlabArgs A)
{
    const int lane = threadIdx.x & 31;
    const int s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (s >= A.nsci) return;
    const int slot0 = 32 * s;
    // column of this slab: last c with col_start[c] <= slot0
    int lo = 0, hi = A.ncol - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (A.col_start[mid] <= slot0) lo = mid; else hi = mid - 1;
    }
    const int c = lo;
    const int r = (slot0 - A.col_start[c]) / 32;
    const int cnt = A.col_count[c];
    const int m = min(32, cnt - 32 * r);
    const bool real = lane < m;
    int idx = 0;
    float3 w = make_float3(0.f, 0.f, 0.f), k = make_float3(0.f, 0.f, 0.f);
    if (real) {
        idx = A.sorted[A.col_astart[c] + 32 * r + lane];
        w = wrap_atom(A.B.x, idx, A.B, k);
    }
    const unsigned long long u = (unsigned long long)(unsigned)idx;
    int r1 = group_rank(((unsigned long long)ordkey(w.y) << 32) | u, 0, real);
    int h = r1 >= 16 ? 1 : 0;
    int r2 = group_rank(((unsigned long long)ordkey(w.x) << 32) | u, h, real);
    int qd = r2 >= 8 ? 1 : 0;
    int r3 = group_rank(((unsigned long long)ordkey(w.z) << 32) | u, 2 * h + qd, real);
    int off = 16 * h + 8 * qd + r3;
    unsigned occ = __reduce_or_sync(0xffffffffu, real ? (1u << off) : 0u);
    if (real) {
        int slot = slot0 + off;
        int g = A.gid_in ? A.gid_in[idx] : idx;
        NBX_DCHECK(g >= 0 && g < A.natoms_global && slot0 + off < 32 * A.nsci);
        float q = A.q_g[g];
        A.order[slot] = idx;
        A.gid[slot] = g;
        A.type[slot] = A.type_g[g];
        A.xq[slot] = make_float4(w.x, w.y, w.z, q);
        A.wrapk[slot] = make_float4(k.x, k.y, k.z, q);
        A.slotmap[g] = slot;
        A.islot[idx] = slot;
    }
    if (!((occ >> lane) & 1u)) {
        int slot = slot0 + lane;
        A.order[slot] = -1;
        A.gid[slot] = -1;
        A.type[slot] = 0;
        A.xq[slot] = make_float4(NBX_FILLER_COORD, NBX_FILLER_COORD, NBX_FILLER_COORD, 0.f);
        A.wrapk[slot] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
}

struct BBArgs {
    int nsci;
    const int* order;
    const int* gid;
    const float4* xq;
    float4* bb_ci;
    float4* bb_cj;
    float4* bb_sci;
    double* sumq2;
};

__device__ __forceinline__ void bb_reduce(float3& lo, float3& hi, int& nr, int x0, int x1)
{
    for (int o = x0; o <= x1; o <<= 1) {
        lo.x = fminf(lo.x, __shfl_xor_sync(0xffffffffu, lo.x, o));
        lo.y = fminf(lo.y, __shfl_xor_sync(0xffffffffu, lo.y, o));
        lo.z = fminf(lo.z, __shfl_xor_sync(0xffffffffu, lo.z, o));
        hi.x = fmaxf(hi.x, __shfl_xor_sync(0xffffffffu, hi.x, o));
        hi.y = fmaxf(hi.y, __shfl_xor_sync(0xffffffffu, hi.y, o));
        hi.z = fmaxf(hi.z, __shfl_xor_sync(0xffffffffu, hi.z, o));
        nr += __shfl_xor_sync(0xffffffffu, nr, o);
    }
}

// grid-stride over super-clusters, one warp each; the fp64 sum of q^2 (self energy) is kept
// per warp and reduced per block, so there is one global atomic per block, not per sci
__global__ void k_bbox(BBArgs A, int gslot)
{
    __shared__ double s_q2;
    const int lane = threadIdx.x & 31;
    if (threadIdx.x == 0) s_q2 = 0.0;
    __syncthreads();
    double q2w = 0.0;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; s < A.nsci; s += nw) {
        const int slot = 32 * s + lane;
        const bool real = A.order[slot] >= 0;
        float4 x = A.xq[slot];
        float3 lo = real ? make_float3(x.x, x.y, x.z) : make_float3(NBX_BB_EMPTY, NBX_BB_EMPTY, NBX_BB_EMPTY);
        float3 hi = real ? make_float3(x.x, x.y, x.z) : make_float3(-NBX_BB_EMPTY, -NBX_BB_EMPTY, -NBX_BB_EMPTY);
        int nr = real ? 1 : 0;
        q2w += real ? (double)x.w * (double)x.w : 0.0;
        bb_reduce(lo, hi, nr, 1, 2);
        if ((lane & 3) == 0) {
            int ci = 8 * s + (lane >> 2);
            A.bb_ci[2 * ci] = make_float4(lo.x, lo.y, lo.z, (float)nr);
            A.bb_ci[2 * ci + 1] = make_float4(hi.x, hi.y, hi.z, 0.f);
        }
        bb_reduce(lo, hi, nr, 4, 4);
        if ((lane & 7) == 0) {
            int cj = 4 * s + (lane >> 3);
            A.bb_cj[2 * cj] = make_float4(lo.x, lo.y, lo.z, (float)nr);
            A.bb_cj[2 * cj + 1] = make_float4(hi.x, hi.y, hi.z, 0.f);
        }
        bb_reduce(lo, hi, nr, 8, 16);
        if (lane == 0) {
            A.bb_sci[2 * s] = make_float4(lo.x, lo.y, lo.z, (float)nr);
            A.bb_sci[2 * s + 1] = make_float4(hi.x, hi.y, hi.z, 0.f);
        }
    }
    for (int o = 16; o > 0; o >>= 1) q2w += __shfl_xor_sync(0xffffffffu, q2w, o);
    if (lane == 0) atomicAdd(&s_q2, q2w);
    __syncthreads();
    if (threadIdx.x == 0) atomicAdd(&A.sumq2[gslot], s_q2);
}

// x-y bounding box of every column (union of its slab boxes), for the search's exact
// column pre-test; empty columns get an empty box
__global__ void k_colbox(int ncol, const int* __restrict__ col_start, const float4* __restrict__ bb_sci,
                         float4* __restrict__ bb_col)
{
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= ncol) return;
    float4 b = make_float4(NBX_BB_EMPTY, NBX_BB_EMPTY, -NBX_BB_EMPTY, -NBX_BB_EMPTY);
    for (int k = col_start[c] >> 5; k < (col_start[c + 1] >> 5); k++) {
        const float4 lo = bb_sci[2 * k], hi = bb_sci[2 * k + 1];
        b.x = fminf(b.x, lo.x);
        b.y = fminf(b.y, lo.y);
        b.z = fmaxf(b.z, hi.x);
        b.w = fmaxf(b.w, hi.y);
    }
    bb_col[c] = b;
}

// host-side grid dimensions: the same formula as ora_grid_dims (oracle/nbx_oracle.c)
static void grid_dims(const float size[3], double density, int* ncx, int* ncy, float inv_cell[2])
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

static int bits_for(int v)
{
    int b = 0;
    while ((1ll << b) <= v) b++;
    return b;
}

// grid build in two halves around the one host read it needs (the padded slot count, which
// sizes every later buffer and launch): grid_begin enqueues binning, the column sort and the
// scans plus an async read into pinned host memory; grid_end, after the caller has waited,
// enqueues the slab fill and the bounding boxes.  grid_build = begin + wait + end;
// grid_build_pair overlaps two grids (DD: home + halo) on two streams with one wait.
static void grid_begin(nbx_ctx* ctx, int g, int n, const float* x, const int* gid, const float lo[3],
                const float size[3], cudaStream_t st, GridStage& S)
{
    Grid& G = ctx->grid[g];
    G.n = n;
    for (int d = 0; d < 3; d++) { G.lo[d] = lo[d]; G.size[d] = size[d]; }
    grid_dims(size, ctx->density, &G.ncx, &G.ncy, G.inv_cell);
    G.ncol = G.ncx * G.ncy;
    const int nn = n > 0 ? n : 1;
    G.col_count.ensure(G.ncol + 1);
    G.col_start.ensure(G.ncol + 1);
    G.col_astart.ensure(G.ncol + 1);
    G.key.ensure(nn); G.key_out.ensure(nn); G.val.ensure(nn); G.val_out.ensure(nn);
    NBX_CUDA(cudaMemsetAsync(G.col_count.p, 0, sizeof(int) * (G.ncol + 1), st));

    BinArgs B;
    B.n = n;
    B.x = x;
    B.box = make_float3(ctx->box[0], ctx->box[1], ctx->box[2]);
    B.invL = make_float3((float)(1.0 / (double)ctx->box[0]), (float)(1.0 / (double)ctx->box[1]),
                         (float)(1.0 / (double)ctx->box[2]));
    B.lo = make_float3(lo[0], lo[1], lo[2]);
    for (int d = 0; d < 3; d++) B.pbc[d] = ctx->pbc[d];
    B.inv_cell[0] = G.inv_cell[0];
    B.inv_cell[1] = G.inv_cell[1];
    B.ncx = G.ncx;
    B.ncy = G.ncy;
    if (n > 0) {
        k_bin<<<(n + 255) / 256, 256, 0, st>>>(B, G.key.p, G.val.p, G.col_count.p);
        ctx->launches++;
        NBX_CUDA(cudaGetLastError());
        size_t tb = 0;
        int endbit = 32 + bits_for(G.ncol);
        NBX_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, G.key.p, G.key_out.p, G.val.p,
                                                 G.val_out.p, n, 0, endbit, st));
        G.tmp.ensure(tb + 16);
        NBX_CUDA(cub::DeviceRadixSort::SortPairs(G.tmp.p, tb, G.key.p, G.key_out.p, G.val.p,
                                                 G.val_out.p, n, 0, endbit, st));
        ctx->launches += 4;
    }
    // padded column sizes -> slot offsets; atom offsets
    int* padded = G.val.p; // reuse (n >= 1); needs ncol+1 ints
    if ((size_t)(G.ncol + 1) > G.val.cap) { G.padded.ensure(G.ncol + 1); padded = G.padded.p; }
    k_pad<<<(G.ncol + 1 + 255) / 256, 256, 0, st>>>(G.col_count.p, G.ncol, padded);
    ctx->launches++;
    size_t tb1 = 0, tb2 = 0;
    NBX_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb1, padded, G.col_start.p, G.ncol + 1, st));
    NBX_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb2, G.col_count.p, G.col_astart.p, G.ncol + 1, st));
    G.tmp.ensure((tb1 > tb2 ? tb1 : tb2) + 16);
    NBX_CUDA(cub::DeviceScan::ExclusiveSum(G.tmp.p, tb1, padded, G.col_start.p, G.ncol + 1, st));
    NBX_CUDA(cub::DeviceScan::ExclusiveSum(G.tmp.p, tb2, G.col_count.p, G.col_astart.p, G.ncol + 1, st));
    ctx->launches += 2;
    S.B = B;
    S.gid = gid;
    S.h = host_pin(ctx) + 4 * g; // [0]: padded slot count
    NBX_CUDA(cudaMemcpyAsync(S.h, G.col_start.p + G.ncol, sizeof(int), cudaMemcpyDeviceToHost, st));
}

static void grid_end(nbx_ctx* ctx, int g, cudaStream_t st, const GridStage& S)
{
    Grid& G = ctx->grid[g];
    const BinArgs& B = S.B;
    const int* gid = S.gid;
    const int n = G.n, nn = n > 0 ? n : 1;
    const int nslots = S.h[0];
    G.nslots = nslots;
    G.nsci = nslots / 32;
    const int ns = nslots > 0 ? nslots : 32;
    G.order.ensure(ns); G.gid.ensure(ns); G.type.ensure(ns);
    G.xq.ensure(ns); G.wrapk.ensure(ns); G.f.ensure(ns);
    G.bb_ci.ensure(2 * (ns / 4)); G.bb_cj.ensure(2 * (ns / 8)); G.bb_sci.ensure(2 * (ns / 32));
    G.slotmap.ensure(ctx->natoms_global + 1);
    G.islot.ensure(nn);
    NBX_CUDA(cudaMemsetAsync(G.slotmap.p, 0xff, sizeof(int) * (ctx->natoms_global + 1), st));
    NBX_CUDA(cudaMemsetAsync(G.f.p, 0, sizeof(float4) * ns, st));
    NBX_CUDA(cudaMemsetAsync(ctx->sumq2.p + g, 0, sizeof(double), st));
    if (G.nsci > 0) {
        SlabArgs S;
        S.B = B;
        S.nsci = G.nsci;
        S.ncol = G.ncol;
        S.col_start = G.col_start.p;
        S.col_astart = G.col_astart.p;
        S.col_count = G.col_count.p;
        S.sorted = G.val_out.p;
        S.gid_in = gid;
        S.q_g = ctx->q_g.p;
        S.type_g = ctx->type_g.p;
        S.order = G.order.p;
        S.gid = G.gid.p;
        S.type = G.type.p;
        S.xq = G.xq.p;
        S.wrapk = G.wrapk.p;
        S.slotmap = G.slotmap.p;
        S.islot = G.islot.p;
        S.natoms_global = ctx->natoms_global;
        int threads = 128, blocks = (G.nsci * 32 + threads - 1) / threads;
        k_slab<<<blocks, threads, 0, st>>>(S);
        ctx->launches++;
        NBX_CUDA(cudaGetLastError());
        BBArgs BA;
        BA.nsci = G.nsci;
        BA.order = G.order.p;
        BA.gid = G.gid.p;
        BA.xq = G.xq.p;
        BA.bb_ci = G.bb_ci.p;
        BA.bb_cj = G.bb_cj.p;
        BA.bb_sci = G.bb_sci.p;
        BA.sumq2 = ctx->sumq2.p;
        const int bblocks = std::min(blocks, ctx->num_sms * 16);
        k_bbox<<<bblocks, threads, 0, st>>>(BA, g);
        ctx->launches++;
        NBX_CUDA(cudaGetLastError());
    }
    G.bb_col.ensure(G.ncol);
    k_colbox<<<(G.ncol + 255) / 256, 256, 0, st>>>(G.ncol, G.col_start.p, G.bb_sci.p, G.bb_col.p);
    ctx->launches++;
    NBX_CUDA(cudaGetLastError());
    G.built = true;
}

void grid_build(nbx_ctx* ctx, int g, int n, const float* x, const int* gid, const float lo[3],
                const float size[3], cudaStream_t st)
{
    GridStage S;
    grid_begin(ctx, g, n, x, gid, lo, size, st, S);
    NBX_CUDA(cudaStreamSynchronize(st));
    grid_end(ctx, g, st, S);
}

void grid_build_pair(nbx_ctx* ctx, const GridReq r[2], cudaStream_t st0, cudaStream_t st1)
{
    GridStage S0, S1;
    grid_begin(ctx, 0, r[0].n, r[0].x, r[0].gid, r[0].lo, r[0].size, st0, S0);
    grid_begin(ctx, 1, r[1].n, r[1].x, r[1].gid, r[1].lo, r[1].size, st1, S1);
    NBX_CUDA(cudaStreamSynchronize(st0));
    NBX_CUDA(cudaStreamSynchronize(st1));
    grid_end(ctx, 0, st0, S0);
    grid_end(ctx, 1, st1, S1);
}

} // namespace nbx
