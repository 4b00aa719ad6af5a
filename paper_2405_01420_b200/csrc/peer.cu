// peer.cu -- the DD halo over NVLink peer memory, one process per GPU.
//
// The reference's halo (pipeline.py:273-278 coordinate pulses, 363-380 pack/unpack, 403-418
// reverse force pulses) is simulated time; the NCCL form of it lives in dd.py.  This file is
// the fused form: no messages, no pack/unpack, no reverse pulses.
//
//   * every rank publishes its home coordinates (xpub, home order) in an IPC-shared region,
//     written by the grid-0 X buffer op itself, then signals "x ready (seq)" to all ranks;
//   * the importer waits for the flags and gathers its halo coordinates straight from the
//     owners' xpub over NVLink into the cluster-ordered grid-1 xyzq (+ the import shift);
//   * the nonlocal force kernel accumulates the halo j forces in the grid-1 cluster buffer and
//     one push kernel red.global.add.v4.f32's each halo atom's force straight into its
//     owner's force inbox (home order) over NVLink, then signals "f done (seq)".  (The fully
//     fused form, k_force<..., REMOTE> sending every j-cluster entry's forces to the owner
//     from the force kernel itself, is kept behind NBX_PEER_FUSED=1: it issues ~10x more
//     remote reductions and measured 0.26 vs 0.16 ms for the 12 M nonlocal kernel at N=2);
//   * the owner waits for those flags and its F buffer op adds the inbox to the home forces
//     (and clears it for the next step).
//
// Flags are per-rank uint32 sequence numbers: rank r's region holds flags[2][world], written
// by rank w with st.release.sys at [kind][w] and spun on with ld.acquire.sys by r.  The spin
// is bounded (NBX_PEER_TIMEOUT_S, default 30 s): a missing peer sets an error word that
// nbx_peer_status reports and then traps, so a timed-out step can never go on to read stale
// or half-written peer memory (the CUDA context is lost and every later call fails loudly).
//
// Energy / virial steps run through the same halo (flags NBX_FORCE_ENERGY / VIRIAL): the
// virial sum x (x) f of the halo atoms is taken on the importing rank from grid 1's cluster
// forces (halo coordinates in this rank's frame) BEFORE they are pushed to the owners, and the
// home atoms' sum from grid 0 BEFORE the inbox is added, so each cross-domain pair enters
// exactly one rank's virial -- the single-sum form of -1/2 sum_pairs r_ij (x) f_ij.
#include <cstdlib>
#include <cstring>

#include "nbx_internal.cuh"

namespace nbx {

struct Peer {
    int rank = 0, world = 0, cap = 0, n_halo = 0;
    char* base = nullptr;        // own IPC region: flags | xpub | inbox
    unsigned* flags = nullptr;   // [2][world]
    float4* xpub = nullptr;      // [cap] home coordinates (x, y, z, 0) of this step
    float4* inbox = nullptr;     // [cap] forces on home atoms from other ranks' nonlocal lists
    std::vector<char*> remote;   // opened peer regions (nullptr for self)
    DBuf<unsigned*> d_flags;     // [world] flag arrays of every rank
    DBuf<float4*> d_xpub, d_inbox;
    DBuf<const float4*> src;     // [n_halo] owner xpub entry of halo input atom a
    DBuf<float4> hshift;         // [n_halo] import shift of halo input atom a
    DBuf<float4*> fj_dst;        // [grid-1 nslots] owner inbox entry (or own padding slot)
    DBuf<float4*> dst;           // [n_halo] owner inbox entry of halo input atom a
    bool fused = false;          // NBX_PEER_FUSED=1: remote j forces from the force kernel
    DBuf<int> err;               // [1] wait timed out
    bool open = false, halo = false;
    unsigned long long timeout_ns = 30ull * 1000000000ull;
};

static size_t flags_bytes(int world) { return ((size_t)2 * world * sizeof(unsigned) + 255) / 256 * 256; }

__device__ __forceinline__ unsigned long long gtimer()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void k_peer_signal(unsigned* const* flags, int world, int slot, unsigned seq)
{
    const int w = threadIdx.x;
    if (w >= world) return;
    __threadfence_system(); // this stream's earlier kernels' writes / reds before the flag
    unsigned* p = flags[w] + slot;
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(seq) : "memory");
}

__global__ void k_peer_wait(const unsigned* flags, int world, int kind, unsigned seq, int* err,
                            unsigned long long timeout_ns)
{
    const int w = threadIdx.x;
    if (w >= world) return;
    const unsigned* p = flags + kind * world + w;
    const unsigned long long t0 = gtimer();
    for (;;) {
        unsigned v;
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
        if ((int)(v - seq) >= 0) break;
        if (gtimer() - t0 > timeout_ns) {
            atomicExch(err, 1);
            __threadfence_system();
            __trap(); // fatal: the step must not consume stale peer memory
        }
        __nanosleep(128);
    }
}

// grid-0 X buffer op that also publishes the home coordinates
__global__ void k_peer_put_x(int nslots, const int* __restrict__ order, const float4* __restrict__ wrapk,
                             const float* __restrict__ x, float3 box, float4* __restrict__ xq,
                             float4* __restrict__ xpub)
{
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= nslots) return;
    const int a = order[s];
    if (a < 0) return;
    const float4 k = wrapk[s];
    const float x0 = x[3 * a], x1 = x[3 * a + 1], x2 = x[3 * a + 2];
    xq[s] = make_float4(__fmaf_rn(-k.x, box.x, x0), __fmaf_rn(-k.y, box.y, x1), __fmaf_rn(-k.z, box.z, x2), k.w);
    xpub[a] = make_float4(x0, x1, x2, 0.0f);
}

// grid-1 X buffer op reading the owners' published coordinates over NVLink
__global__ void k_peer_halo_x(int nslots, const int* __restrict__ order, const float4* __restrict__ wrapk,
                              float3 box, const float4* const* __restrict__ src,
                              const float4* __restrict__ hshift, float4* __restrict__ xq)
{
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= nslots) return;
    const int a = order[s];
    if (a < 0) return;
    const float4 k = wrapk[s];
    const float4 v = __ldcv(src[a]);
    const float4 h = hshift[a];
    const float x0 = __fadd_rn(v.x, h.x), x1 = __fadd_rn(v.y, h.y), x2 = __fadd_rn(v.z, h.z);
    xq[s] = make_float4(__fmaf_rn(-k.x, box.x, x0), __fmaf_rn(-k.y, box.y, x1), __fmaf_rn(-k.z, box.z, x2), k.w);
}

// grid-0 F buffer op + the forces other ranks put into this rank's inbox (cleared after use)
__global__ void k_peer_get_f(int n, const int* __restrict__ islot, const float4* __restrict__ fc,
                             float4* __restrict__ inbox, float* __restrict__ f)
{
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= n) return;
    const float4 v = fc[islot[a]];
    const float4 r = __ldcg(inbox + a);
    inbox[a] = make_float4(0.f, 0.f, 0.f, 0.f);
    f[3 * a] = v.x + r.x;
    f[3 * a + 1] = v.y + r.y;
    f[3 * a + 2] = v.z + r.z;
}

// halo forces -> owners' inboxes: one remote v4 reduction per imported atom
__global__ void k_peer_push(int n, const int* __restrict__ islot, const float4* __restrict__ fc,
                            float4* const* __restrict__ dst)
{
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= n) return;
    const float4 v = fc[islot[a]];
    red_add_v4(dst[a], make_float4(v.x, v.y, v.z, 0.f));
}

__global__ void k_peer_src(int n, const int* __restrict__ owner, const int* __restrict__ home,
                           const float* __restrict__ shift, float4* const* xpub, float4* const* inbox,
                           const float4** src, float4** dst, float4* hshift)
{
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= n) return;
    src[a] = xpub[owner[a]] + home[a];
    dst[a] = inbox[owner[a]] + home[a];
    hshift[a] = make_float4(shift[3 * a], shift[3 * a + 1], shift[3 * a + 2], 0.f);
}

__global__ void k_peer_dst(int nslots, const int* __restrict__ order, const int* __restrict__ owner,
                           const int* __restrict__ home, float4* const* inbox, float4* local_f, float4** dst)
{
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= nslots) return;
    const int a = order[s];
    dst[s] = (a < 0) ? local_f + s : inbox[owner[a]] + home[a];
}

static Peer& need(nbx_ctx* ctx, bool want_open, bool want_halo)
{
    Peer* P = ctx->peer;
    if (!P) throw CudaError{cudaErrorInvalidValue, "peer halo not initialised (nbx_peer_init)"};
    if (want_open && !P->open) throw CudaError{cudaErrorInvalidValue, "peer regions not opened (nbx_peer_open)"};
    if (want_halo && !P->halo) throw CudaError{cudaErrorInvalidValue, "peer halo map not set (nbx_peer_set_halo)"};
    return *P;
}

void peer_release(nbx_ctx* ctx)
{
    Peer* P = ctx->peer;
    if (!P) return;
    for (char* r : P->remote)
        if (r) cudaIpcCloseMemHandle(r);
    if (P->base) cudaFree(P->base);
    P->d_flags.release(); P->d_xpub.release(); P->d_inbox.release(); P->src.release();
    P->hshift.release(); P->fj_dst.release(); P->dst.release(); P->err.release();
    delete P;
    ctx->peer = nullptr;
}

void peer_init(nbx_ctx* ctx, int rank, int world, int cap, void* handle_out)
{
    peer_release(ctx);
    Peer* P = new Peer;
    ctx->peer = P;
    P->rank = rank;
    P->world = world;
    P->cap = cap;
    if (const char* t = std::getenv("NBX_PEER_TIMEOUT_S")) P->timeout_ns = (unsigned long long)(std::atof(t) * 1e9);
    if (const char* f = std::getenv("NBX_PEER_FUSED")) P->fused = std::atoi(f) != 0;
    const size_t fb = flags_bytes(world), bytes = fb + 2 * (size_t)cap * sizeof(float4);
    NBX_CUDA(cudaMalloc((void**)&P->base, bytes));
    NBX_CUDA(cudaMemset(P->base, 0, bytes));
    P->flags = reinterpret_cast<unsigned*>(P->base);
    P->xpub = reinterpret_cast<float4*>(P->base + fb);
    P->inbox = P->xpub + cap;
    P->err.ensure(1);
    NBX_CUDA(cudaMemset(P->err.p, 0, sizeof(int)));
    cudaIpcMemHandle_t h;
    NBX_CUDA(cudaIpcGetMemHandle(&h, P->base));
    static_assert(sizeof(h) == NBX_PEER_HANDLE_BYTES, "IPC handle size");
    std::memcpy(handle_out, &h, sizeof(h));
    NBX_CUDA(cudaDeviceSynchronize());
}

void peer_open(nbx_ctx* ctx, const void* handles)
{
    Peer& P = need(ctx, false, false);
    const size_t fb = flags_bytes(P.world);
    P.remote.assign(P.world, nullptr);
    std::vector<unsigned*> fl(P.world);
    std::vector<float4*> xp(P.world), ib(P.world);
    for (int w = 0; w < P.world; w++) {
        char* b = P.base;
        if (w != P.rank) {
            cudaIpcMemHandle_t h;
            std::memcpy(&h, static_cast<const char*>(handles) + (size_t)w * sizeof(h), sizeof(h));
            NBX_CUDA(cudaIpcOpenMemHandle((void**)&b, h, cudaIpcMemLazyEnablePeerAccess));
            P.remote[w] = b;
        }
        fl[w] = reinterpret_cast<unsigned*>(b);
        xp[w] = reinterpret_cast<float4*>(b + fb);
        ib[w] = xp[w] + P.cap;
    }
    P.d_flags.ensure(P.world);
    P.d_xpub.ensure(P.world);
    P.d_inbox.ensure(P.world);
    NBX_CUDA(cudaMemcpy(P.d_flags.p, fl.data(), sizeof(unsigned*) * P.world, cudaMemcpyHostToDevice));
    NBX_CUDA(cudaMemcpy(P.d_xpub.p, xp.data(), sizeof(float4*) * P.world, cudaMemcpyHostToDevice));
    NBX_CUDA(cudaMemcpy(P.d_inbox.p, ib.data(), sizeof(float4*) * P.world, cudaMemcpyHostToDevice));
    P.open = true;
}

void peer_set_halo(nbx_ctx* ctx, int n, const int* owner, const int* home, const float* shift, cudaStream_t st)
{
    Peer& P = need(ctx, true, false);
    Grid& G0 = ctx->grid[0];
    Grid& G1 = ctx->grid[1];
    if (!G0.built || !G1.built) throw CudaError{cudaErrorInvalidValue, "build both grids before nbx_peer_set_halo"};
    if (G1.n != n) throw CudaError{cudaErrorInvalidValue, "n_halo differs from the grid-1 atom count"};
    if (G0.n > P.cap) throw CudaError{cudaErrorInvalidValue, "home atoms exceed the peer capacity"};
    P.n_halo = n;
    NBX_CUDA(cudaMemsetAsync(P.err.p, 0, sizeof(int), st));
    P.src.ensure(n > 0 ? n : 1);
    P.dst.ensure(n > 0 ? n : 1);
    P.hshift.ensure(n > 0 ? n : 1);
    P.fj_dst.ensure(G1.nslots > 0 ? G1.nslots : 1);
    if (n > 0) {
        k_peer_src<<<(n + 255) / 256, 256, 0, st>>>(n, owner, home, shift, P.d_xpub.p, P.d_inbox.p, P.src.p,
                                                     P.dst.p, P.hshift.p);
        ctx->launches++;
        NBX_CUDA(cudaGetLastError());
    }
    if (P.fused && G1.nslots > 0) {
        k_peer_dst<<<(G1.nslots + 255) / 256, 256, 0, st>>>(G1.nslots, G1.order.p, owner, home, P.d_inbox.p,
                                                            G1.f.p, P.fj_dst.p);
        ctx->launches++;
        NBX_CUDA(cudaGetLastError());
    }
    P.halo = true;
}

static void signal(nbx_ctx* ctx, Peer& P, int kind, unsigned seq, cudaStream_t st)
{
    k_peer_signal<<<1, 32 * ((P.world + 31) / 32), 0, st>>>(P.d_flags.p, P.world, kind * P.world + P.rank, seq);
    ctx->launches++;
    NBX_CUDA(cudaGetLastError());
}

static void wait(nbx_ctx* ctx, Peer& P, int kind, unsigned seq, cudaStream_t st)
{
    k_peer_wait<<<1, 32 * ((P.world + 31) / 32), 0, st>>>(P.flags, P.world, kind, seq, P.err.p, P.timeout_ns);
    ctx->launches++;
    NBX_CUDA(cudaGetLastError());
}

void peer_put_x(nbx_ctx* ctx, const float* x, unsigned seq, cudaStream_t st)
{
    Peer& P = need(ctx, true, true);
    Grid& G = ctx->grid[0];
    if (G.nslots > 0) {
        k_peer_put_x<<<(G.nslots + 255) / 256, 256, 0, st>>>(G.nslots, G.order.p, G.wrapk.p, x,
                                                             make_float3(ctx->box[0], ctx->box[1], ctx->box[2]),
                                                             G.xq.p, P.xpub);
        ctx->launches++;
        NBX_CUDA(cudaGetLastError());
    }
    signal(ctx, P, 0, seq, st);
}

void peer_halo_x(nbx_ctx* ctx, unsigned seq, cudaStream_t st)
{
    Peer& P = need(ctx, true, true);
    wait(ctx, P, 0, seq, st);
    Grid& G = ctx->grid[1];
    if (G.nslots > 0) {
        k_peer_halo_x<<<(G.nslots + 255) / 256, 256, 0, st>>>(G.nslots, G.order.p, G.wrapk.p,
                                                              make_float3(ctx->box[0], ctx->box[1], ctx->box[2]),
                                                              P.src.p, P.hshift.p, G.xq.p);
        ctx->launches++;
        NBX_CUDA(cudaGetLastError());
    }
}

void peer_force_nonlocal(nbx_ctx* ctx, unsigned seq, unsigned flags, cudaStream_t st)
{
    Peer& P = need(ctx, true, true);
    Grid& G = ctx->grid[1];
    if (P.fused && !flags) {
        if (ctx->list[1].built && ctx->list[1].n_sci > 0) force(ctx, 1, 0, st, P.fj_dst.p);
    } else {
        if (ctx->list[1].built && ctx->list[1].n_sci > 0) force(ctx, 1, flags, st);
        if (flags & NBX_FORCE_VIRIAL) {
            // halo atoms' x (x) f while their forces are still here (section header)
            virial_sum(ctx, 1, st);
            ctx->xf_done |= 2;
        }
        if (G.n > 0) {
            k_peer_push<<<(G.n + 255) / 256, 256, 0, st>>>(G.n, G.islot.p, G.f.p, P.dst.p);
            ctx->launches++;
            NBX_CUDA(cudaGetLastError());
        }
        if (G.nslots > 0) NBX_CUDA(cudaMemsetAsync(G.f.p, 0, sizeof(float4) * G.nslots, st));
    }
    signal(ctx, P, 1, seq, st);
}

void peer_get_f(nbx_ctx* ctx, float* f, unsigned seq, unsigned flags, cudaStream_t st)
{
    Peer& P = need(ctx, true, true);
    if (flags & NBX_FORCE_VIRIAL) {
        // home atoms' x (x) f from the forces computed on this rank (local + nonlocal lists),
        // before the inbox (pairs other ranks computed and count) is added
        virial_sum(ctx, 0, st);
        ctx->xf_done |= 1;
    }
    wait(ctx, P, 1, seq, st);
    Grid& G = ctx->grid[0];
    if (G.n > 0) {
        k_peer_get_f<<<(G.n + 255) / 256, 256, 0, st>>>(G.n, G.islot.p, G.f.p, P.inbox, f);
        ctx->launches++;
        NBX_CUDA(cudaGetLastError());
    }
    if (G.nslots > 0) NBX_CUDA(cudaMemsetAsync(G.f.p, 0, sizeof(float4) * G.nslots, st));
}

int peer_status(nbx_ctx* ctx)
{
    Peer& P = need(ctx, false, false);
    int e = 0;
    NBX_CUDA(cudaMemcpy(&e, P.err.p, sizeof(int), cudaMemcpyDeviceToHost));
    return e;
}

} // namespace nbx
