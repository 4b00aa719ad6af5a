// nbx_internal.cuh -- context, device buffers and shared helpers of libnbx (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <cufft.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/nbx.h"

#define NBX_FILLER_COORD (-1.0e5f)
#define NBX_BB_EMPTY 1.0e30f
#define NBX_R2MIN 1.0e-6f
// dynamic shared memory opted into by the force kernels (LJ table + EWALD_TAB tables);
// nbx_set_topology rejects tables that would not fit
#define FORCE_SMEM_MAX (96 * 1024)

namespace nbx {

void set_error(const std::string& msg);
int fail(int code, const std::string& msg);

struct CudaError {
    cudaError_t err;
    const char* what;
};

// Checked builds (-DNBX_CHECKED=1, tools/checked_build.py): every data-dependent index the
// kernels read from lists, grids or caller arrays is range-checked on the device, and a
// violation fails a device assert (the stand-in for compute-sanitizer memcheck,
// which this GPU pool does not run).  Compiled out of the shipped library.
#ifndef NBX_CHECKED
#define NBX_CHECKED 0
#endif
#if NBX_CHECKED
#undef NDEBUG
#include <cassert>
// device assert: the failed condition (tagged NBX_DCHECK) is printed and the kernel stops with
// cudaErrorAssert, which every later call on the context reports
#define NBX_DCHECK(cond) assert((cond) && "NBX_DCHECK")
#else
#define NBX_DCHECK(cond) \
    do {                 \
    } while (0)
#endif

#define NBX_CUDA(call)                                                               \
    do {                                                                             \
        cudaError_t _e = (call);                                                     \
        if (_e != cudaSuccess) throw ::nbx::CudaError{_e, #call};                     \
    } while (0)

// device allocations made by DBuf::ensure (process-wide; nbx_alloc_count).  cudaMalloc and
// cudaFree take the driver's resource-manager lock, which an nvidia-smi / NVML poll also
// holds: an allocation inside a step can stall it by a poll interval (measured: 12 M DD search
// steps 12 -> 45-270 ms with nvidia-smi sampling at 250 ms).  Steady-state steps allocate
// nothing: buffers grow with 12.5 % headroom and scratch buffers are kept.
extern unsigned long long g_allocs;
extern int g_trace_allocs; // env NBX_TRACE_ALLOCS=1: log every allocation to stderr
void trace_alloc(size_t bytes, size_t old_bytes, void* caller);

// Grow-only device buffer.
template <class T>
struct DBuf {
    T* p = nullptr;
    size_t cap = 0;
    void ensure(size_t n)
    {
        if (n <= cap && p) return;
        if (p) NBX_CUDA(cudaFree(p));
        p = nullptr;
        size_t want = n < 16 ? 16 : n + n / 8;
        NBX_CUDA(cudaMalloc((void**)&p, want * sizeof(T)));
        __atomic_add_fetch(&g_allocs, 1ull, __ATOMIC_RELAXED);
        if (g_trace_allocs) trace_alloc(want * sizeof(T), cap * sizeof(T), __builtin_return_address(0));
        cap = want;
    }
    void release()
    {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
};

struct Grid {
    int n = 0, nslots = 0, nsci = 0, ncx = 0, ncy = 0, ncol = 0;
    float lo[3] = {0, 0, 0}, size[3] = {0, 0, 0}, inv_cell[2] = {0, 0};
    bool built = false;
    DBuf<int> col_count, col_start, col_astart; // [ncol], [ncol+1], [ncol+1]
    DBuf<unsigned long long> key, key_out;      // sort keys [n]
    DBuf<int> val, val_out;                     // sort values [n]
    DBuf<float4> xw;                            // wrapped coords + ... per input atom [n]
    DBuf<int> order, gid, type;                 // [nslots]
    DBuf<float4> xq;                            // [nslots] x,y,z,q
    DBuf<float4> wrapk;                         // [nslots] kx,ky,kz,q
    DBuf<float4> f;                             // [nslots] cluster forces (w unused)
    DBuf<float4> bb_ci, bb_cj, bb_sci;          // 2 float4 per cluster: lo (w = nreal), hi
    DBuf<float4> bb_col;                        // per column: (xlo, ylo, xhi, yhi) of its atoms
    DBuf<int> slotmap;                          // global id -> slot, or -1 [natoms_global]
    DBuf<int> islot;                            // input index -> slot [n]
    DBuf<int> padded;                           // padded column sizes [ncol + 1] (when val is too small)
    DBuf<char> tmp;                             // cub temp
};

struct List {
    int64_t n_sci = 0, n_cj = 0, n_pool = 0;
    bool built = false;
    int gi = 0, gj = 0, mode = 0;
    DBuf<nbx_sci_entry> sci, sci_in;
    DBuf<nbx_cj_entry> cj, cj_in;
    DBuf<nbx_mask_pool_entry> pool;
    DBuf<int> counts;  // [3][nsci+1]
    DBuf<int> offsets; // [3][nsci+1]
    DBuf<int> totals;  // [3]
    DBuf<unsigned> len_key, len_key_out;        // force-kernel work order (row f2)
    DBuf<int> order_in, order;                  // sci entries, longest first
    bool use_order = false;                     // order is valid and the force kernel uses it
    DBuf<char> sort_tmp;
    DBuf<int> flags;                            // search overflow / max counts
    DBuf<unsigned long long> pair_count;        // nbx_count_pairs scratch [2]
    int cap_cj = 0, cap_pool = 0;               // single-pass per-sci capacities
    DBuf<nbx_sci_entry> tsci;                   // single-pass private outputs
    DBuf<nbx_cj_entry> tcj;
    DBuf<nbx_mask_pool_entry> tpool;
    DBuf<char> tmp;
    int prune_chunks = 0;            // split prune: 32-entry chunks of the longest sci (0: off)
    DBuf<nbx_cj_entry> prune_tmp;    // split prune: per-chunk compacted entries [n_cj]
    DBuf<int> prune_kept;            // split prune: kept count per (entry, chunk)
};

struct Peer; // peer.cu: NVLink peer-memory halo state (DD, row e)

struct ForceConsts {
    float epsfac, k_rf, two_k_rf, c_rf, beta, beta2, beta3, beta3_monic, sh_ewald, sh_lj6, sh_lj12, rc2, rli2;
    float fsw_r1, fsw_a6, fsw_b6, fsw_a12, fsw_b12, fsw_p6, fsw_q6, fsw_p12, fsw_q12, fsw_c6, fsw_c12;
    float tab_scale;
    float rc2_big;   // rc2 * 2^64: cut-off step as one FFMA.SAT (force-only kernels)
    unsigned one;    // 1, opaque to the compiler: integer adds issued as IMAD (FMA pipe)
    float ewn[6], ewd[5]; // F-only Ewald: -beta^3 G as N(r2) / D(r2), D monic (pairmath.cuh)
    alignas(8) float ewnd[10]; // (ewn[k], ewd[k]) interleaved: one 64-bit constant per FFMA2
    alignas(8) float ehnd[12]; // energy kernels' H(z) rational: (num, den) coefficient pairs
    alignas(8) float ehbd[12]; // NBX_VF_H: the same with the numerator scaled by beta (beta H)
    float ehb0, two_sh_lj6;    // beta * H's last numerator coefficient; 2 sh_lj6
};

} // namespace nbx

struct nbx_ctx {
    int device = 0;
    int num_sms = 148;
    nbx_params p{};
    nbx_consts c{};
    int natoms_global = 0, ntypes = 0;
    bool have_topology = false, have_box = false;
    float box[3] = {0, 0, 0};
    int pbc[3] = {1, 1, 1};
    double density = 0.0;
    nbx::DBuf<float> q_g;
    nbx::DBuf<int> type_g;
    nbx::DBuf<int> excl_off_g, excl_gid_g;
    nbx::DBuf<float2> c6c12s; // (6 c6, 12 c12)
    nbx::DBuf<float2> ewtab;  // EWALD_TAB: [tab_n] (F, dF) then [tab_n] (V, dV)
    nbx::Grid grid[2];
    nbx::List list[2];
    nbx::DBuf<double> acc;    // [0..1] E_lj, E_coul ; [2..82] fshift ; [83..91] sum x (x) f
    nbx::DBuf<double> sumq2;  // [2] per grid
    nbx::DBuf<int> counter;   // work counters [8]
    int64_t launches = 0;
    int force_split = 0; // > 0: fixed work items per sci entry (env NBX_FORCE_SPLIT), 0: auto
    int prune_split = -1; // split prune for short lists: -1 auto, 0 off, 1 on (env NBX_PRUNE_SPLIT)
    int prune_kernel = 2; // 0: k_prune (lane per cj entry), 1: k_prune_lanes (lane per i atom), 2: k_prune_packed (compacted tiles, FP32x2); env NBX_PRUNE_KERNEL
    // row f2, force-kernel work order: 0 = list order (spatially coherent), 1 = longest entry
    // first (sorted after every prune), -1 = auto (default): longest first for lists of
    // 1,024 <= n_sci < 32 x the resident force warps, where the tail matters and L2 locality
    // does not yet (measured: mem82k -7.5 %, STMV -1.8 % force kernel; 12 M +5 %, water 3k's
    // ~10 us sort is not repaid), analytical Ewald / RF only (tabulated Ewald: +2.9 %).
    // Env NBX_ENTRY_ORDER overrides.
    int entry_order = -1;
    // nbx_step_graph: natively captured X op (+ prune) + force + F op, one per (x, f, what);
    // `epoch` is bumped by every call that can move list/grid buffers or change constants,
    // and a stale graph is refreshed with cudaGraphExecUpdate (no re-instantiation).
    struct StepGraph {
        const float* x;
        float* f;
        uint32_t what;
        uint64_t epoch;
        int kernels;
        cudaGraphExec_t exec;
    };
    nbx::Peer* peer = nullptr;
    // peer-halo energy steps: x (x) f already summed per grid (bit 0: grid 0, bit 1: grid 1)
    // by nbx_peer_get_f / nbx_peer_force_nonlocal, so nbx_energies must not re-sum it
    unsigned xf_done = 0;
    uint64_t epoch = 1;
    std::vector<StepGraph> graphs;
    // nbx_step_graph_pme: the same plus PME on grid 0 and the leap-frog update, keyed by all
    // buffers, the PME context (and its epoch) and dt
    struct FullGraph {
        const void* pme;
        uint64_t pme_epoch;
        const float* x;
        float* f;
        float* v;
        const float* inv_mass;
        float dt;
        uint32_t what;
        uint64_t epoch;
        int kernels;
        cudaGraphExec_t exec;
    };
    std::vector<FullGraph> full_graphs;
    cudaStream_t cap_stream = nullptr;
    // pinned host words for the search step's size reads (async copies; grid g at [4 g],
    // list l at [8 + 8 l])
    int* h_pin = nullptr;
    cudaEvent_t ev_pair[2] = {nullptr, nullptr}; // nbx_grid_search_pair stream ordering
};

namespace nbx {
inline int* host_pin(nbx_ctx* ctx)
{
    if (!ctx->h_pin) NBX_CUDA(cudaMallocHost((void**)&ctx->h_pin, 32 * sizeof(int)));
    return ctx->h_pin;
}
} // namespace nbx

// PME context (row f4; pme.cu)
struct nbx_pme {
    int device = 0;
    int nk[3] = {0, 0, 0};
    float beta = 0.f, epsfac = 0.f;
    float box[3] = {0.f, 0.f, 0.f};
    bool have_box = false;
    nbx::DBuf<float> grid;    // real grid [nx][ny][nz]: charges, then the potential
    nbx::DBuf<float2> spec;   // half spectrum [nx][ny][nz/2+1]
    nbx::DBuf<float> bmod;    // |b(m)|^2: [nx] then [ny] then [nz/2+1]
    nbx::DBuf<float> gex;     // exp(-pi^2 mt_d^2 / beta^2), same layout (set_box)
    nbx::DBuf<double> acc;    // [0] energy, [1..9] virial
    cufftHandle fwd = 0, inv = 0;
    int64_t launches = 0;
    uint64_t epoch = 1; // bumped by set_box (graph refresh)
};

namespace nbx {

// ---- shared device helpers ------------------------------------------------------------
__device__ __forceinline__ uint32_t ordkey(float f)
{
    uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__device__ __forceinline__ void red_add_v4(float4* p, float4 v)
{
    asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y),
                 "f"(v.z), "f"(v.w)
                 : "memory");
}

// predicated v4 reduction (no branch / reconvergence around the lanes that write)
__device__ __forceinline__ void red_add_v4_if(float4* p, float4 v, unsigned cond)
{
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %5, 0;\n\t@q red.global.add.v4.f32 [%0], {%1,%2,%3,%4};\n\t}"
                 ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(cond)
                 : "memory");
}

// shift vector of shift index s (0..26): exactly (float)sx * box[d] as in the oracle
__device__ __forceinline__ float3 shift_vec(int s, float3 box)
{
    int sx = s % 3 - 1, sy = (s / 3) % 3 - 1, sz = s / 9 - 1;
    return make_float3(__fmul_rn((float)sx, box.x), __fmul_rn((float)sy, box.y),
                       __fmul_rn((float)sz, box.z));
}

// ---- launchers (defined in the .cu files) -----------------------------------------------
struct GridReq {
    int n;
    const float* x;
    const int* gid;
    const float* lo;
    const float* size;
};
// grids 0 and 1 built concurrently on st0 / st1 with one host wait (DD search steps)
void grid_build_pair(nbx_ctx* ctx, const GridReq r[2], cudaStream_t st0, cudaStream_t st1);
// lists 0 and 1 searched concurrently on st0 / st1 with one host wait; st1 must already be
// ordered after grid 0's build (list 1's i grid), st0 is not ordered after st1 on return
void search_pair(nbx_ctx* ctx, cudaStream_t st0, cudaStream_t st1);
void grid_build(nbx_ctx* ctx, int g, int n, const float* x, const int* gid, const float lo[3],
                const float size[3], cudaStream_t st);
void search(nbx_ctx* ctx, int l, cudaStream_t st);
void prune(nbx_ctx* ctx, int l, int part, int nparts, cudaStream_t st);
void count_pairs(nbx_ctx* ctx, int l, long long* pairs, long long* slots, cudaStream_t st);
void force(nbx_ctx* ctx, int l, unsigned flags, cudaStream_t st, float4* const* fj_dst = nullptr);
void put_x(nbx_ctx* ctx, int g, const float* x, cudaStream_t st);
void get_f(nbx_ctx* ctx, int g, float* f, int accumulate, cudaStream_t st);
void virial_sum(nbx_ctx* ctx, int g, cudaStream_t st);
void halo_pack_x(const float* x, const int* idx, int n, float3 shift, float* out, cudaStream_t st);
void halo_unpack_add_f(float* f, const int* idx, int n, const float* in, cudaStream_t st);
double fma_peak(cudaStream_t st);
void peer_release(nbx_ctx* ctx);
void peer_init(nbx_ctx* ctx, int rank, int world, int cap, void* handle_out);
void peer_open(nbx_ctx* ctx, const void* handles);
void peer_set_halo(nbx_ctx* ctx, int n, const int* owner, const int* home, const float* shift, cudaStream_t st);
void peer_put_x(nbx_ctx* ctx, const float* x, unsigned seq, cudaStream_t st);
void peer_halo_x(nbx_ctx* ctx, unsigned seq, cudaStream_t st);
void peer_force_nonlocal(nbx_ctx* ctx, unsigned seq, unsigned flags, cudaStream_t st);
void peer_get_f(nbx_ctx* ctx, float* f, unsigned seq, unsigned flags, cudaStream_t st);
int peer_status(nbx_ctx* ctx);
int peer_repartition(nbx_ctx* ctx, const nbx_dd_geom* g, const float* xh, const int* gh, int nh, unsigned rseq,
                     int cap_ext, float* x_ext, int* gid_ext, int* owner, int* home, float* shift, int* nh_out,
                     int* nhalo_out, cudaStream_t st);
ForceConsts make_force_consts(const nbx_consts& c);
void pme_setup(nbx_pme* pme);
void pme_set_box(nbx_pme* pme, const float box[3]);
void pme_compute(nbx_pme* pme, int n, const float* x, const float* q, float* f, unsigned flags, cudaStream_t st,
                 cudaEvent_t* ev = nullptr, bool xq4 = false);
void pme_compute_grid(nbx_pme* pme, nbx_ctx* ctx, int grid, unsigned flags, cudaStream_t st);
void pme_profile(nbx_pme* pme, int n, const float* x, const float* q, float* f, float ms[6], cudaStream_t st);
void pme_energy(nbx_pme* pme, double* e, double* vir, cudaStream_t st);
void pme_release(nbx_pme* pme);
void leapfrog(int n, float* x, float* v, const float* f, const float* inv_mass, float dt, cudaStream_t st);

} // namespace nbx
