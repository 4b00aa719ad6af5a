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

#include <cub/device/device_radix_sort.cuh>

#include "nbx_internal.cuh"

namespace nbx {

struct Peer {
    int rank = 0, world = 0, cap = 0, n_halo = 0;
    char* base = nullptr;        // own IPC region: flags | counts | xpub | inbox | xpub2 | gpub | gpub2
    unsigned* flags = nullptr;   // [4][world]: x ready, f done, homes published, new homes published
    int* cnt = nullptr;          // [0] published home count, [1] published new-home count
    float4* xpub = nullptr;      // [cap] home coordinates (x, y, z, 0) of this step
    float4* inbox = nullptr;     // [cap] forces on home atoms from other ranks' nonlocal lists
    float4* xpub2 = nullptr;     // [cap] repartition: the new home atoms (wrapped x, sorted by gid)
    int* gpub = nullptr;         // [cap] repartition: global ids of the published home atoms
    int* gpub2 = nullptr;        // [cap] repartition: global ids of the new home atoms
    DBuf<float4*> d_xpub2;       // [world] every rank's xpub2 / gpub / gpub2 / cnt
    DBuf<int*> d_gpub, d_gpub2, d_cnt;
    DBuf<int> rp_key, rp_key_out, rp_val, rp_val_out, rp_cnt; // repartition scratch
    DBuf<float4> rp_stage;
    DBuf<char> rp_tmp;
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

static size_t flags_bytes(int world) { return ((size_t)4 * world * sizeof(unsigned) + 255) / 256 * 256; }
constexpr size_t CNT_BYTES = 256;
// byte offsets of the region's arrays (identical on every rank: same world and cap)
struct PeerLayout {
    size_t flags, cnt, xpub, inbox, xpub2, gpub, gpub2, bytes;
    PeerLayout(int world, int cap)
    {
        const size_t c16 = (size_t)cap * sizeof(float4), c4 = ((size_t)cap * sizeof(int) + 255) / 256 * 256;
        flags = 0;
        cnt = flags_bytes(world);
        xpub = cnt + CNT_BYTES;
        inbox = xpub + c16;
        xpub2 = inbox + c16;
        gpub = xpub2 + c16;
        gpub2 = gpub + c4;
        bytes = gpub2 + c4;
    }
};

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
                             float4* __restrict__ xpub, int cap)
{
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= nslots) return;
    const int a = order[s];
    if (a < 0) return;
    NBX_DCHECK(a < cap);
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
    NBX_DCHECK(islot[a] >= 0);
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
    float4* d = dst[a];
    if (d) red_add_v4(d, make_float4(v.x, v.y, v.z, 0.f)); // null: an invalid map entry (err 2)
}

__global__ void k_peer_src(int n, const int* __restrict__ owner, const int* __restrict__ home,
                           const float* __restrict__ shift, float4* const* xpub, float4* const* inbox,
                           const float4** src, float4** dst, float4* hshift, int world, int cap, int* err)
{
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= n) return;
    if (owner[a] < 0 || owner[a] >= world || home[a] < 0 || home[a] >= cap) {
        // a halo map pointing outside the peer regions: never dereference it (the step's
        // gather / push would read or reduce into foreign memory); nbx_peer_status reports 2
        atomicExch(err, 2);
        src[a] = xpub[0];
        dst[a] = nullptr;
        hshift[a] = make_float4(0.f, 0.f, 0.f, 0.f);
        return;
    }
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
    P->d_xpub2.release(); P->d_gpub.release(); P->d_gpub2.release(); P->d_cnt.release();
    P->rp_key.release(); P->rp_key_out.release(); P->rp_val.release(); P->rp_val_out.release();
    P->rp_cnt.release(); P->rp_stage.release(); P->rp_tmp.release();
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
    const PeerLayout Lo(world, cap);
    NBX_CUDA(cudaMalloc((void**)&P->base, Lo.bytes));
    NBX_CUDA(cudaMemset(P->base, 0, Lo.bytes));
    P->flags = reinterpret_cast<unsigned*>(P->base + Lo.flags);
    P->cnt = reinterpret_cast<int*>(P->base + Lo.cnt);
    P->xpub = reinterpret_cast<float4*>(P->base + Lo.xpub);
    P->inbox = reinterpret_cast<float4*>(P->base + Lo.inbox);
    P->xpub2 = reinterpret_cast<float4*>(P->base + Lo.xpub2);
    P->gpub = reinterpret_cast<int*>(P->base + Lo.gpub);
    P->gpub2 = reinterpret_cast<int*>(P->base + Lo.gpub2);
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
    const PeerLayout Lo(P.world, P.cap);
    P.remote.assign(P.world, nullptr);
    std::vector<unsigned*> fl(P.world);
    std::vector<float4*> xp(P.world), ib(P.world), xp2(P.world);
    std::vector<int*> gp(P.world), gp2(P.world), cn(P.world);
    for (int w = 0; w < P.world; w++) {
        char* b = P.base;
        if (w != P.rank) {
            cudaIpcMemHandle_t h;
            std::memcpy(&h, static_cast<const char*>(handles) + (size_t)w * sizeof(h), sizeof(h));
            NBX_CUDA(cudaIpcOpenMemHandle((void**)&b, h, cudaIpcMemLazyEnablePeerAccess));
            P.remote[w] = b;
        }
        fl[w] = reinterpret_cast<unsigned*>(b + Lo.flags);
        cn[w] = reinterpret_cast<int*>(b + Lo.cnt);
        xp[w] = reinterpret_cast<float4*>(b + Lo.xpub);
        ib[w] = reinterpret_cast<float4*>(b + Lo.inbox);
        xp2[w] = reinterpret_cast<float4*>(b + Lo.xpub2);
        gp[w] = reinterpret_cast<int*>(b + Lo.gpub);
        gp2[w] = reinterpret_cast<int*>(b + Lo.gpub2);
    }
    P.d_flags.ensure(P.world);
    P.d_xpub.ensure(P.world);
    P.d_inbox.ensure(P.world);
    P.d_xpub2.ensure(P.world);
    P.d_gpub.ensure(P.world);
    P.d_gpub2.ensure(P.world);
    P.d_cnt.ensure(P.world);
    NBX_CUDA(cudaMemcpy(P.d_flags.p, fl.data(), sizeof(unsigned*) * P.world, cudaMemcpyHostToDevice));
    NBX_CUDA(cudaMemcpy(P.d_xpub.p, xp.data(), sizeof(float4*) * P.world, cudaMemcpyHostToDevice));
    NBX_CUDA(cudaMemcpy(P.d_inbox.p, ib.data(), sizeof(float4*) * P.world, cudaMemcpyHostToDevice));
    NBX_CUDA(cudaMemcpy(P.d_xpub2.p, xp2.data(), sizeof(float4*) * P.world, cudaMemcpyHostToDevice));
    NBX_CUDA(cudaMemcpy(P.d_gpub.p, gp.data(), sizeof(int*) * P.world, cudaMemcpyHostToDevice));
    NBX_CUDA(cudaMemcpy(P.d_gpub2.p, gp2.data(), sizeof(int*) * P.world, cudaMemcpyHostToDevice));
    NBX_CUDA(cudaMemcpy(P.d_cnt.p, cn.data(), sizeof(int*) * P.world, cudaMemcpyHostToDevice));
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
                                                     P.dst.p, P.hshift.p, P.world, P.cap, P.err.p);
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
                                                             G.xq.p, P.xpub, P.cap);
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

// ---- device-side repartition (nbx_peer_repartition; include/nbx.h) -----------------------
// Phase A: publish the current home atoms (x, gid, count), signal kind 2, wait for everyone,
// pull from the neighbour ranks the atoms whose wrapped position lies in this domain, sort
// them by global id (deterministic home order), publish them as the new home set (xpub2,
// gpub2), signal kind 3.  Phase B: wait, pull the half-shell halo from the neighbours' new
// home sets, sort by (offset, owner home index).  The wrap and domain arithmetic is the host
// path's (dd.py repartition: xw = x - floor(x / L) L, c = floor(xw / D) clamped) in IEEE
// single precision, so every rank decides every atom's owner identically: each atom lands in
// exactly one new home set (dd.py checks the total).  Kind-2 publication reuses xpub, which
// nobody reads any more (every rank passed its previous step's "f done" wait); the new home
// set goes to xpub2, which no rank overwrites before everyone has pulled its halo from it
// (kind-3 wait before the next repartition's publication... many steps later).
constexpr unsigned RP_SENTINEL = 0x7f7f7f7fu; // sorts after every real key (memset byte 0x7f)

__global__ void k_rp_publish(int n, const int* __restrict__ n_dev, int cap, const float* __restrict__ x,
                             const int* __restrict__ gid, float4* __restrict__ xpub, int* __restrict__ gpub,
                             int* __restrict__ cnt, int slot)
{
    const int nn = n_dev ? min(*n_dev, cap) : n;
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a == 0) cnt[slot] = nn;
    if (a >= nn) return;
    xpub[a] = make_float4(x[3 * a], x[3 * a + 1], x[3 * a + 2], 0.0f);
    gpub[a] = gid[a];
}

__device__ __forceinline__ float rp_wrap(float x, float L)
{
    return __fsub_rn(x, __fmul_rn(floorf(__fdiv_rn(x, L)), L));
}

__global__ void k_rp_pull_home(nbx_dd_geom G, const float4* const* __restrict__ xpub, const int* const* __restrict__ gpub,
                               int* const* __restrict__ cnt, int cap, int* __restrict__ counter,
                               int* __restrict__ key, int* __restrict__ val, float4* __restrict__ stage)
{
    const int r = G.src_rank[blockIdx.y];
    const int n = __ldcg(cnt[r]);
    NBX_DCHECK(r >= 0 && n >= 0 && n <= cap); // every rank publishes at most the common capacity
    for (int a = blockIdx.x * blockDim.x + threadIdx.x; a < n; a += gridDim.x * blockDim.x) {
        const float4 p = __ldcg(xpub[r] + a);
        const float w0 = rp_wrap(p.x, G.box[0]), w1 = rp_wrap(p.y, G.box[1]), w2 = rp_wrap(p.z, G.box[2]);
        const float w[3] = {w0, w1, w2};
        bool mine = true;
#pragma unroll
        for (int d = 0; d < 3; d++) {
            int c = (int)floorf(__fdiv_rn(w[d], G.dlen[d]));
            c = c < 0 ? 0 : (c > G.dims[d] - 1 ? G.dims[d] - 1 : c);
            mine = mine && (c == G.coord[d]);
        }
        if (!mine) continue;
        const int slot = atomicAdd(counter, 1);
        if (slot >= cap) continue; // overflow: reported through the count
        key[slot] = __ldcg(gpub[r] + a);
        val[slot] = slot;
        stage[slot] = make_float4(w0, w1, w2, 0.0f);
    }
}

__global__ void k_rp_gather_home(int cap, const int* __restrict__ counter, const int* __restrict__ key,
                                 const int* __restrict__ val, const float4* __restrict__ stage,
                                 float* __restrict__ x, int* __restrict__ gid)
{
    const int n = min(*counter, cap);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const float4 p = stage[val[i]];
        x[3 * i] = p.x;
        x[3 * i + 1] = p.y;
        x[3 * i + 2] = p.z;
        gid[i] = key[i];
    }
}

__global__ void k_rp_pull_halo(nbx_dd_geom G, const float4* const* __restrict__ xpub2,
                               const int* const* __restrict__ gpub2, int* const* __restrict__ cnt, int cap,
                               int* __restrict__ counter, int* __restrict__ key, int* __restrict__ val,
                               float4* __restrict__ stage)
{
    const int oi = blockIdx.y;
    const int r = G.off_rank[oi];
    const int n = __ldcg(cnt[r] + 1);
    NBX_DCHECK(r >= 0 && n >= 0 && n < (1 << 26)); // the home index fits the 26-bit key field
    for (int a = blockIdx.x * blockDim.x + threadIdx.x; a < n; a += gridDim.x * blockDim.x) {
        const float4 p = __ldcg(xpub2[r] + a);
        const float x[3] = {__fadd_rn(p.x, G.off_shift[oi][0]), __fadd_rn(p.y, G.off_shift[oi][1]),
                            __fadd_rn(p.z, G.off_shift[oi][2])};
        bool in = true;
#pragma unroll
        for (int d = 0; d < 3; d++) {
            const int o = G.off_dir[oi][d];
            if (o > 0) in = in && x[d] < __fadd_rn(G.hi[d], G.rl);
            if (o < 0) in = in && x[d] >= __fsub_rn(G.lo[d], G.rl);
        }
        if (!in) continue;
        const int slot = atomicAdd(counter, 1);
        if (slot >= cap) continue;
        key[slot] = (oi << 26) | a;
        val[slot] = slot;
        stage[slot] = make_float4(x[0], x[1], x[2], __int_as_float(__ldcg(gpub2[r] + a)));
    }
}

__global__ void k_rp_gather_halo(nbx_dd_geom G, int cap_ext, const int* __restrict__ counters, int cap_home,
                                 const int* __restrict__ key, const int* __restrict__ val,
                                 const float4* __restrict__ stage, float* __restrict__ x, int* __restrict__ gid,
                                 int* __restrict__ owner, int* __restrict__ home, float* __restrict__ shift)
{
    const int nh = min(counters[0], cap_home);
    const int n = min(counters[1], cap_ext - nh);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const float4 p = stage[val[i]];
        const int k = key[i], oi = k >> 26;
        const int e = nh + i;
        x[3 * e] = p.x;
        x[3 * e + 1] = p.y;
        x[3 * e + 2] = p.z;
        gid[e] = __float_as_int(p.w);
        owner[i] = G.off_rank[oi];
        home[i] = k & ((1 << 26) - 1);
        shift[3 * i] = G.off_shift[oi][0];
        shift[3 * i + 1] = G.off_shift[oi][1];
        shift[3 * i + 2] = G.off_shift[oi][2];
    }
}

static void rp_sort(nbx_ctx* ctx, Peer& P, int n, int end_bit, cudaStream_t st)
{
    size_t tb = 0;
    NBX_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, P.rp_key.p, P.rp_key_out.p, P.rp_val.p, P.rp_val_out.p, n,
                                             0, end_bit, st));
    P.rp_tmp.ensure(tb + 16);
    NBX_CUDA(cub::DeviceRadixSort::SortPairs(P.rp_tmp.p, tb, P.rp_key.p, P.rp_key_out.p, P.rp_val.p,
                                             P.rp_val_out.p, n, 0, end_bit, st));
    ctx->launches += 4;
}

int peer_repartition(nbx_ctx* ctx, const nbx_dd_geom* g, const float* xh, const int* gh, int nh, unsigned rseq,
                     int cap_ext, float* x_ext, int* gid_ext, int* owner, int* home, float* shift, int* nh_out,
                     int* nhalo_out, cudaStream_t st)
{
    Peer& P = need(ctx, true, false);
    if (nh > P.cap) throw CudaError{cudaErrorInvalidValue, "home atoms exceed the peer capacity"};
    if (cap_ext < 1 || cap_ext >= (1 << 26) || P.cap >= (1 << 26))
        throw CudaError{cudaErrorInvalidValue, "repartition capacity out of range (< 2^26)"};
    if (g->n_src < 1 || g->n_src > 27 || g->n_off < 0 || g->n_off > 13)
        throw CudaError{cudaErrorInvalidValue, "bad repartition geometry"};
    const int capw = P.cap > cap_ext ? P.cap : cap_ext;
    P.rp_key.ensure(capw);
    P.rp_key_out.ensure(capw);
    P.rp_val.ensure(capw);
    P.rp_val_out.ensure(capw);
    P.rp_stage.ensure(capw);
    P.rp_cnt.ensure(4);
    NBX_CUDA(cudaMemsetAsync(P.rp_cnt.p, 0, 4 * sizeof(int), st));
    const int T = 256, B = 4 * ctx->num_sms;
    // phase A
    k_rp_publish<<<(nh + T) / T, T, 0, st>>>(nh, nullptr, P.cap, xh, gh, P.xpub, P.gpub, P.cnt, 0);
    ctx->launches++;
    NBX_CUDA(cudaGetLastError());
    signal(ctx, P, 2, rseq, st);
    wait(ctx, P, 2, rseq, st);
    NBX_CUDA(cudaMemsetAsync(P.rp_key.p, 0x7f, sizeof(int) * (size_t)P.cap, st));
    k_rp_pull_home<<<dim3(B, g->n_src), T, 0, st>>>(*g, P.d_xpub.p, P.d_gpub.p, P.d_cnt.p, P.cap, P.rp_cnt.p,
                                                     P.rp_key.p, P.rp_val.p, P.rp_stage.p);
    ctx->launches++;
    NBX_CUDA(cudaGetLastError());
    rp_sort(ctx, P, P.cap, 31, st);
    k_rp_gather_home<<<B, T, 0, st>>>(P.cap < cap_ext ? P.cap : cap_ext, P.rp_cnt.p, P.rp_key_out.p,
                                      P.rp_val_out.p, P.rp_stage.p, x_ext, gid_ext);
    ctx->launches++;
    NBX_CUDA(cudaGetLastError());
    k_rp_publish<<<(P.cap + T - 1) / T, T, 0, st>>>(0, P.rp_cnt.p, P.cap < cap_ext ? P.cap : cap_ext, x_ext, gid_ext,
                                                    P.xpub2, P.gpub2, P.cnt, 1);
    ctx->launches++;
    NBX_CUDA(cudaGetLastError());
    signal(ctx, P, 3, rseq, st);
    // phase B
    wait(ctx, P, 3, rseq, st);
    if (g->n_off > 0) {
        NBX_CUDA(cudaMemsetAsync(P.rp_key.p, 0x7f, sizeof(int) * (size_t)cap_ext, st));
        k_rp_pull_halo<<<dim3(B, g->n_off), T, 0, st>>>(*g, P.d_xpub2.p, P.d_gpub2.p, P.d_cnt.p, cap_ext,
                                                         P.rp_cnt.p + 1, P.rp_key.p, P.rp_val.p, P.rp_stage.p);
        ctx->launches++;
        NBX_CUDA(cudaGetLastError());
        rp_sort(ctx, P, cap_ext, 31, st);
        k_rp_gather_halo<<<B, T, 0, st>>>(*g, cap_ext, P.rp_cnt.p, P.cap, P.rp_key_out.p, P.rp_val_out.p,
                                          P.rp_stage.p, x_ext, gid_ext, owner, home, shift);
        ctx->launches++;
        NBX_CUDA(cudaGetLastError());
    }
    int h[2] = {0, 0};
    NBX_CUDA(cudaMemcpyAsync(h, P.rp_cnt.p, sizeof(h), cudaMemcpyDeviceToHost, st));
    NBX_CUDA(cudaStreamSynchronize(st));
    *nh_out = h[0];
    *nhalo_out = h[1];
    return (h[0] > P.cap || h[0] + h[1] > cap_ext) ? 1 : 0;
}

int peer_status(nbx_ctx* ctx)
{
    Peer& P = need(ctx, false, false);
    int e = 0;
    NBX_CUDA(cudaMemcpy(&e, P.err.p, sizeof(int), cudaMemcpyDeviceToHost));
    return e;
}

} // namespace nbx
