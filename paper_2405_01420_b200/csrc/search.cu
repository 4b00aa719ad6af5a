// search.cu -- cluster-pair search (KernelKind.PAIR_SEARCH, costs.py:32,163; pipeline.py:226-230)
// and the rolling dynamic prune (KernelKind.PRUNE_ONLY, costs.py:31,162; pipeline.py:233-235).
//
// Search: one warp per super-cluster.  Per shift image, the warp enumerates the candidate
// grid columns 32 at a time (one binary search over the column's z-sorted slabs per lane,
// all in flight together; columns whose x-y box is out of range are dropped by an exact
// pre-test), prefix-sums their j-cluster counts and tests the candidates in two phases: one
// candidate per lane against the super-cluster bounding box (survivors and their boxes go to
// a per-warp shared-memory table), then the survivors' 8 i-cluster tiles spread over the
// lanes (lane = survivor * 8 + i-cluster), all at rlist_outer.  Explicit masks are computed
// only for tiles that contain an excluded partner (each i-atom's partners are mapped to their
// j-cluster through the grid's gid -> slot map into a per-warp shared-memory list, behind an
// exact 64-bit filter), contain filler slots or lie on the diagonal (the nonlocal list has no
// diagonal: every home x halo pair is computed there) -- by the whole warp, one tile per pass,
// one atom pair per lane.  The list is written deterministically at ballot/popc ranks -- the
// canonical (sci, shift, cj) order of the CPU oracle (ora_search), bit for bit: in one pass
// into per-sci private regions (capacity learned from the previous search) plus a
// compaction, or, for the first search and on overflow, a count pass, exclusive scans and a
// fill pass.
//
// Prune (default k_prune_packed): one warp per sci entry; per 32-entry chunk the active tiles
// are compacted into an item table; a row sweep (one lane per tile, i atom 1 against the 8 j
// atoms) keeps about half of them, and the rest are tested 8 per warp pass (4 lanes per tile,
// packed FP32x2 r^2 at rlist_inner); kept entries are compacted in order.  Short lists use the split
// form (a warp per chunk + a gather).  k_prune / k_prune_lanes / k_prune_fixed are opt-ins.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "f32x2.cuh"
#include "nbx_internal.cuh"

namespace nbx {

constexpr int SEARCH_THREADS = 128;
#ifndef NBX_SEARCH_V2
// 1: phase B takes the i-cluster and survivor boxes from shared memory (staged once per sci /
// per candidate chunk) and evaluates explicit tile masks cooperatively -- one tile per warp
// pass, one atom pair per lane -- instead of 32 pairs serially in the owning lane
#define NBX_SEARCH_V2 1
#endif
constexpr int EXMAX = 24; // partner j-clusters remembered per i-cluster (overflow -> always check)

struct SearchArgs {
    // i grid
    const float4* bb_ci;
    const float4* bb_sci;
    const int* order_i;
    const int* gid_i;
    int nsci_i;
    // j grid
    const float4* bb_cj;
    const float4* bb_sci_j;
    const int* order_j;
    const int* gid_j;
    const int* slotmap_j; // global id -> slot in grid j, or -1
    const int* col_start_j;
    const float4* bb_col_j; // (xlo, ylo, xhi, yhi) per column
    int ncx_j, ncy_j;
    float lo_jx, lo_jy, inv_jx, inv_jy;
    // topology
    const int* excl_off;
    const int* excl_gid;
    float3 box;
    int pbc0, pbc1, pbc2;
    int mode;
    float rl, rl2, rlm;
    // outputs
    int* counts;        // [3][nsci+1]
    const int* offsets; // [3][nsci+1]
    nbx_sci_entry* sci_out;
    nbx_cj_entry* cj_out;
    nbx_mask_pool_entry* pool_out;
    // single pass: per-sci private regions of capacity cap_cj / cap_pool, compacted afterwards
    int cap_cj, cap_pool;
    int* flags; // [0] overflow, [1] max n_cj per sci, [2] max n_pool per sci
    int ncl_j;  // j clusters in grid j (checked builds)
};

enum { SEARCH_COUNT = 0, SEARCH_FILL = 1, SEARCH_SINGLE = 2 };

struct WarpEx {
    int cj[8][EXMAX];
    int n[8];
    unsigned long long pbits[8]; // per i-cluster: bit (cj & 63) set for every partner j-cluster
    int surv[32]; // candidates that passed the super-cluster test, in candidate order
#if NBX_SEARCH_V2
    float4 sbb[32][2]; // their bounding boxes (lo, hi), so phase B re-reads nothing global
    float4 ibb[8][2];  // the super-cluster's 8 i-cluster boxes (unshifted)
#endif
};

__device__ __forceinline__ float bb_dist2(float4 alo, float4 ahi, float3 v, float4 blo, float4 bhi)
{
    float ax0 = __fadd_rn(alo.x, v.x), ax1 = __fadd_rn(ahi.x, v.x);
    float ay0 = __fadd_rn(alo.y, v.y), ay1 = __fadd_rn(ahi.y, v.y);
    float az0 = __fadd_rn(alo.z, v.z), az1 = __fadd_rn(ahi.z, v.z);
    float dx = fmaxf(0.0f, fmaxf(__fsub_rn(ax0, bhi.x), __fsub_rn(blo.x, ax1)));
    float dy = fmaxf(0.0f, fmaxf(__fsub_rn(ay0, bhi.y), __fsub_rn(blo.y, ay1)));
    float dz = fmaxf(0.0f, fmaxf(__fsub_rn(az0, bhi.z), __fsub_rn(blo.z, az1)));
    return __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
}

// interaction / exclusion-correction masks of tile (ci, cj), DESIGN.md "Masks"
__device__ uint2 tile_masks(const SearchArgs& A, int ci, int cj, bool exov, bool central)
{
    uint32_t im = 0u, cm = 0u;
    for (int i = 0; i < 4; i++) {
        const int a = 4 * ci + i;
        if (A.order_i[a] < 0) continue;
        const int ga = A.gid_i[a];
        const int e0 = exov ? A.excl_off[ga] : 0, e1 = exov ? A.excl_off[ga + 1] : 0;
        for (int j = 0; j < 8; j++) {
            const int b = 8 * cj + j;
            if (A.order_j[b] < 0) continue;
            const int gb = A.gid_j[b];
            const bool present = (A.mode == NBX_LIST_LOCAL) ? !(central && b <= a) : true;
            if (!present) continue;
            bool ex = false;
            for (int e = e0; e < e1; e++) ex |= (A.excl_gid[e] == gb);
            const uint32_t bit = 1u << (i * 8 + j);
            if (ex) cm |= bit; else im |= bit;
        }
    }
    return make_uint2(im, cm);
}

__device__ __forceinline__ bool has_partner(const WarpEx& X, int k, int cj)
{
    // exact negative filter: a j-cluster whose bit is clear is no partner (the list scan below
    // runs for partners and ~1 in 16 others)
    if (!((X.pbits[k] >> (cj & 63)) & 1ull)) return false;
    const int n = X.n[k];
    if (n > EXMAX) return true;
    bool hit = false;
    for (int m = 0; m < n; m++) hit |= (X.cj[k][m] == cj);
    return hit;
}

// bit u of the result = (byte u of b != 0): OR-fold each byte into its bit 0, then gather the
// four bits with one multiply (the partial products land on distinct bits, no carries)
__device__ __forceinline__ unsigned byte_any4(unsigned b)
{
    b |= b >> 1;
    b |= b >> 2;
    b |= b >> 4;
    return ((b & 0x01010101u) * 0x01020408u) >> 24;
}

// super-cluster level test of one candidate j-cluster
__device__ __forceinline__ bool sci_test(const SearchArgs& A, int sci, int cj, float3 v, bool central,
                                         float4 slo, float4 shi)
{
    if (A.mode == NBX_LIST_LOCAL && central && cj < 4 * sci) return false;
    const float4 blo = A.bb_cj[2 * cj], bhi = A.bb_cj[2 * cj + 1];
    if (blo.w == 0.0f) return false;
    return bb_dist2(slo, shi, v, blo, bhi) < A.rl2;
}

// one (i-cluster k, j-cluster cj) tile of a surviving candidate: (0,0) if it is not in the
// list, (~0, 0) for a plain tile, explicit masks for filler / diagonal / nonlocal /
// excluded-partner tiles
__device__ __forceinline__ uint2 tile_eval(const SearchArgs& A, const WarpEx& X, int sci, int k, int cj,
                                           float3 v, bool central)
{
    const int ci = 8 * sci + k;
    const float4 ilo = A.bb_ci[2 * ci], ihi = A.bb_ci[2 * ci + 1];
    const float4 blo = A.bb_cj[2 * cj], bhi = A.bb_cj[2 * cj + 1];
    if (ilo.w == 0.0f || !(bb_dist2(ilo, ihi, v, blo, bhi) < A.rl2)) return make_uint2(0u, 0u);
    const bool exov = has_partner(X, k, cj);
    const bool masked = ilo.w < 4.0f || blo.w < 8.0f || (central && (cj >> 2) == sci) || exov;
    if (!masked) return make_uint2(0xffffffffu, 0u);
    const uint2 m = tile_masks(A, ci, cj, exov, central);
    return ((m.x | m.y) != 0u) ? m : make_uint2(0u, 0u);
}

// explicit masks of tile (ci, cj) by the whole warp: lane = atom pair (i = lane / 8, j = lane % 8),
// whose bit is i * 8 + j = lane -- the same bits tile_masks() builds in one lane
__device__ __forceinline__ uint2 tile_masks_warp(const SearchArgs& A, int ci, int cj, bool exov, bool central,
                                                 int lane)
{
    const int a = 4 * ci + (lane >> 3), b = 8 * cj + (lane & 7);
    bool ok = A.order_i[a] >= 0 && A.order_j[b] >= 0;
    if (A.mode == NBX_LIST_LOCAL && central && b <= a) ok = false;
    bool ex = false;
    if (ok && exov) {
        const int ga = A.gid_i[a], gb = A.gid_j[b];
        const int e1 = A.excl_off[ga + 1];
        for (int e = A.excl_off[ga]; e < e1; e++) ex |= (A.excl_gid[e] == gb);
    }
    const unsigned FULL = 0xffffffffu;
    return make_uint2(__ballot_sync(FULL, ok && !ex), __ballot_sync(FULL, ok && ex));
}

template <int MODE>
#ifndef NBX_SEARCH_MINB
// 12 CTAs/SM (<= 42 registers, 48 warps): grid + search + prune of a search step 12 M 19.6 ->
// 16.1 ms, STMV 2.58 -> 2.30 ms (RNase 24k +7 %, its search is launch-bound); 1 (64 registers)
// was round 1's (profiles/r02_search_variants.jsonl)
#define NBX_SEARCH_MINB 12
#endif
__global__ void __launch_bounds__(SEARCH_THREADS, NBX_SEARCH_MINB) k_search(SearchArgs A)
{
    __shared__ WarpEx s_ex[SEARCH_THREADS / 32];
    const int lane = threadIdx.x & 31;
    const int sci = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (sci >= A.nsci_i) return;
    WarpEx& X = s_ex[threadIdx.x >> 5];
    const unsigned FULL = 0xffffffffu;
    const unsigned lt = (1u << lane) - 1u;

    // excluded partners of the 32 atoms -> their j-clusters in grid j, per i-cluster
    if (lane < 8) {
        X.n[lane] = 0;
        X.pbits[lane] = 0ull;
    }
    __syncwarp();
    {
        const int slot = 32 * sci + lane;
        if (A.order_i[slot] >= 0) {
            const int g = A.gid_i[slot];
            for (int e = A.excl_off[g]; e < A.excl_off[g + 1]; e++) {
                const int sp = A.slotmap_j[A.excl_gid[e]];
                if (sp >= 0) {
                    const int pos = atomicAdd(&X.n[lane >> 2], 1);
                    if (pos < EXMAX) X.cj[lane >> 2][pos] = sp >> 3;
                    atomicOr(&X.pbits[lane >> 2], 1ull << ((sp >> 3) & 63));
                }
            }
        }
    }
#if NBX_SEARCH_V2
    if (lane < 16) X.ibb[lane >> 1][lane & 1] = A.bb_ci[2 * (8 * sci) + lane];
#endif
    __syncwarp();

    const float4 slo = A.bb_sci[2 * sci], shi = A.bb_sci[2 * sci + 1];
    int n_ent = 0, n_cj = 0, n_pool = 0;
    int ent_base = 0, cj_base = 0, pool_base = 0;
    if (MODE == SEARCH_FILL) {
        ent_base = A.offsets[sci];
        cj_base = A.offsets[(A.nsci_i + 1) + sci];
        pool_base = 1 + A.offsets[2 * (A.nsci_i + 1) + sci];
    } else if (MODE == SEARCH_SINGLE) {
        ent_base = NBX_NSHIFT * sci;
        cj_base = A.cap_cj * sci;
        pool_base = A.cap_pool * sci; // private pool slots, 1-based local index stored in meta
    }
    constexpr bool WRITE = MODE != SEARCH_COUNT;
    if (slo.w != 0.0f) {
        for (int s = 0; s < NBX_NSHIFT; s++) {
            const int sx = s % 3 - 1, sy = (s / 3) % 3 - 1, sz = s / 9 - 1;
            if ((!A.pbc0 && sx) || (!A.pbc1 && sy) || (!A.pbc2 && sz)) continue;
            if (A.mode == NBX_LIST_LOCAL && s < NBX_CENTRAL_SHIFT) continue;
            const bool central = (s == NBX_CENTRAL_SHIFT);
            const float3 v = shift_vec(s, A.box);
            const float lx = __fadd_rn(slo.x, v.x), hx = __fadd_rn(shi.x, v.x);
            const float ly = __fadd_rn(slo.y, v.y), hy = __fadd_rn(shi.y, v.y);
            const float lz = __fadd_rn(slo.z, v.z), hz = __fadd_rn(shi.z, v.z);
            int cx0 = (int)floorf((lx - A.rl - A.lo_jx) * A.inv_jx) - 1;
            int cx1 = (int)floorf((hx + A.rl - A.lo_jx) * A.inv_jx) + 1;
            int cy0 = (int)floorf((ly - A.rl - A.lo_jy) * A.inv_jy) - 1;
            int cy1 = (int)floorf((hy + A.rl - A.lo_jy) * A.inv_jy) + 1;
            cx0 = max(cx0, 0);
            cy0 = max(cy0, 0);
            cx1 = min(cx1, A.ncx_j - 1);
            cy1 = min(cy1, A.ncy_j - 1);
            if (cx1 < cx0 || cy1 < cy0) continue;
            const float zlo = lz - A.rlm, zhi = hz + A.rlm;
            const int nyr = cy1 - cy0 + 1;
            const int ncols = (cx1 - cx0 + 1) * nyr;
            const int start_cj = n_cj;
            for (int cb = 0; cb < ncols; cb += 32) {
                // one column per lane: slab range by two binary searches (monotone z bounds)
                const int ci_ = cb + lane;
                int ks = 0, nc = 0;
                int col = -1;
                if (ci_ < ncols) {
                    col = (cx0 + ci_ / nyr) * A.ncy_j + (cy0 + ci_ % nyr);
                    // exact pre-test: every j-cluster of the column lies inside the column's x-y
                    // box, and fp add/sub/max/fma are monotone, so d2(column) <= d2(any cj)
                    const float4 cb_ = A.bb_col_j[col];
                    const float ddx = fmaxf(0.0f, fmaxf(__fsub_rn(lx, cb_.z), __fsub_rn(cb_.x, hx)));
                    const float ddy = fmaxf(0.0f, fmaxf(__fsub_rn(ly, cb_.w), __fsub_rn(cb_.y, hy)));
                    if (!(__fmaf_rn(ddy, ddy, __fmul_rn(ddx, ddx)) < A.rl2)) col = -1;
                }
                if (col >= 0) {
                    const int k0 = A.col_start_j[col] >> 5, k1 = A.col_start_j[col + 1] >> 5;
                    int a = k0, b = k1;
                    while (a < b) {
                        const int mid = (a + b) >> 1;
                        if (A.bb_sci_j[2 * mid + 1].z < zlo) a = mid + 1; else b = mid;
                    }
                    ks = a;
                    b = k1;
                    while (a < b) {
                        const int mid = (a + b) >> 1;
                        if (A.bb_sci_j[2 * mid].z > zhi) b = mid; else a = mid + 1;
                    }
                    nc = 4 * (a - ks);
                }
                int incl = nc;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int t = __shfl_up_sync(FULL, incl, o);
                    if (lane >= o) incl += t;
                }
                const int excl = incl - nc;
                const int total = __shfl_sync(FULL, incl, 31);
                for (int tb = 0; tb < total; tb += 32) {
                    const int t = tb + lane;
                    int own = 0;
#pragma unroll
                    for (int st = 16; st > 0; st >>= 1) {
                        const int c = own + st;
                        const int ec = __shfl_sync(FULL, excl, c & 31);
                        if (c < 32 && ec <= t) own = c;
                    }
                    const int base_o = __shfl_sync(FULL, excl, own);
                    const int ks_o = __shfl_sync(FULL, ks, own);
                    const int cj = 4 * ks_o + (t - base_o);
                    // phase A: one candidate per lane against the super-cluster box
#if NBX_SEARCH_V2
                    bool pass = (t < total) && !(A.mode == NBX_LIST_LOCAL && central && cj < 4 * sci);
                    float4 blo = make_float4(0.f, 0.f, 0.f, 0.f), bhi = blo;
                    if (pass) {
                        NBX_DCHECK(cj >= 0 && cj < A.ncl_j);
                        blo = A.bb_cj[2 * cj];
                        bhi = A.bb_cj[2 * cj + 1];
                        pass = blo.w != 0.0f && bb_dist2(slo, shi, v, blo, bhi) < A.rl2;
                    }
                    const unsigned S = __ballot_sync(FULL, pass);
                    if (pass) {
                        const int r = __popc(S & lt);
                        X.surv[r] = cj;
                        X.sbb[r][0] = blo;
                        X.sbb[r][1] = bhi;
                    }
#else
                    const bool pass = (t < total) && sci_test(A, sci, cj, v, central, slo, shi);
                    const unsigned S = __ballot_sync(FULL, pass);
                    if (pass) X.surv[__popc(S & lt)] = cj;
#endif
                    __syncwarp();
                    const int ns = __popc(S);
                    // phase B: lane = (survivor q0 + lane/8, i-cluster lane%8), 4 survivors per pass
                    const int sub = lane >> 3, k = lane & 7;
                    const unsigned sublt = (1u << sub) - 1u;
                    for (int q0 = 0; q0 < ns; q0 += 4) {
                        const int q = q0 + sub;
                        const int cjq = (q < ns) ? X.surv[q] : 0;
#if NBX_SEARCH_V2
                        uint2 m = make_uint2(0u, 0u);
                        bool masked = false, exov = false;
                        if (q < ns) {
                            const float4 ilo = X.ibb[k][0], ihi = X.ibb[k][1];
                            const float4 blo = X.sbb[q][0], bhi = X.sbb[q][1];
                            if (ilo.w != 0.0f && bb_dist2(ilo, ihi, v, blo, bhi) < A.rl2) {
                                exov = has_partner(X, k, cjq);
                                masked = ilo.w < 4.0f || blo.w < 8.0f || (central && (cjq >> 2) == sci) || exov;
                                if (!masked) m = make_uint2(0xffffffffu, 0u);
                            }
                        }
                        // tiles that need explicit masks: one per warp pass, a pair per lane
                        unsigned mq = __ballot_sync(FULL, masked);
                        const unsigned xq = __ballot_sync(FULL, exov);
                        while (mq) {
                            const int src = __ffs(mq) - 1;
                            mq &= mq - 1u;
                            const int tcj = __shfl_sync(FULL, cjq, src);
                            const uint2 mm = tile_masks_warp(A, 8 * sci + (src & 7), tcj, (xq >> src) & 1u, central, lane);
                            if (lane == src) m = mm;
                        }
#else
                        const uint2 m = (q < ns) ? tile_eval(A, X, sci, k, cjq, v, central) : make_uint2(0u, 0u);
#endif
                        const bool act = (m.x | m.y) != 0u;
                        const bool need = act && (m.x != 0xffffffffu || m.y != 0u);
                        const unsigned ab = __ballot_sync(FULL, act);
                        const unsigned nb = __ballot_sync(FULL, need);
                        // per survivor (byte u of the ballots): entry emitted / needs a pool entry
                        const unsigned am = byte_any4(ab), pm = byte_any4(nb);
                        if (WRITE && ((am >> sub) & 1u)) {
                            const int cpos = n_cj + __popc(am & sublt);
                            const int ppos = n_pool + __popc(pm & sublt);
                            const bool fits = MODE != SEARCH_SINGLE || (cpos < A.cap_cj && ppos < A.cap_pool);
                            if (fits) {
                                unsigned pidx = 0u;
                                if ((pm >> sub) & 1u) {
                                    pidx = (MODE == SEARCH_SINGLE) ? (unsigned)(ppos + 1) : (unsigned)(pool_base + ppos);
                                    nbx_mask_pool_entry* pe = A.pool_out + (MODE == SEARCH_SINGLE ? pool_base + ppos : pool_base + ppos);
                                    pe->m[k][0] = m.x;
                                    pe->m[k][1] = m.y;
                                }
                                if (k == 0) {
                                    nbx_cj_entry e;
                                    e.cj = cjq;
                                    e.meta = ((ab >> (8 * sub)) & 0xffu) | (pidx << 8);
                                    A.cj_out[cj_base + cpos] = e;
                                }
                            } else if (k == 0) {
                                A.flags[0] = 1;
                            }
                        }
                        n_cj += __popc(am);
                        n_pool += __popc(pm);
                    }
                    __syncwarp();
                }
            }
            if (n_cj > start_cj) {
                if (WRITE && lane == 0) {
                    nbx_sci_entry e;
                    e.sci = sci;
                    e.shift = s;
                    e.cj_start = cj_base + start_cj;
                    e.cj_end = cj_base + n_cj;
                    A.sci_out[ent_base + n_ent] = e;
                }
                n_ent++;
            }
        }
    }
    if (MODE != SEARCH_FILL && lane == 0) {
        A.counts[sci] = n_ent;
        A.counts[(A.nsci_i + 1) + sci] = n_cj;
        A.counts[2 * (A.nsci_i + 1) + sci] = n_pool;
        atomicMax(&A.flags[1], n_cj);
        atomicMax(&A.flags[2], n_pool);
    }
}

// single pass: move each super-cluster's private output to its scanned position and turn the
// local pool indices into global ones
__global__ void k_compact(int nsci, const int* __restrict__ counts, const int* __restrict__ offsets, int cap_cj,
                          int cap_pool, const nbx_sci_entry* __restrict__ tsci, const nbx_cj_entry* __restrict__ tcj,
                          const nbx_mask_pool_entry* __restrict__ tpool, nbx_sci_entry* __restrict__ sci_out,
                          nbx_cj_entry* __restrict__ cj_out, nbx_mask_pool_entry* __restrict__ pool_out)
{
    const int lane = threadIdx.x & 31;
    const int sci = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (sci >= nsci) return;
    const int n1 = nsci + 1;
    const int ne = counts[sci], nc = counts[n1 + sci], np = counts[2 * n1 + sci];
    const int eb = offsets[sci], cb = offsets[n1 + sci], pb = 1 + offsets[2 * n1 + sci];
    const int src_c = cap_cj * sci;
    if (lane < ne) {
        nbx_sci_entry e = tsci[NBX_NSHIFT * sci + lane];
        e.cj_start += cb - src_c;
        e.cj_end += cb - src_c;
        sci_out[eb + lane] = e;
    }
    for (int q = lane; q < nc; q += 32) {
        nbx_cj_entry e = tcj[src_c + q];
        const unsigned pl = e.meta >> 8;
        if (pl) e.meta = (e.meta & 0xffu) | ((unsigned)(pb + pl - 1) << 8);
        cj_out[cb + q] = e;
    }
    const uint4* ps = reinterpret_cast<const uint4*>(tpool + (size_t)cap_pool * sci);
    uint4* pd = reinterpret_cast<uint4*>(pool_out + pb);
    for (int w = lane; w < 4 * np; w += 32) pd[w] = ps[w];
}

__global__ void k_pool0(nbx_mask_pool_entry* pool)
{
    int t = threadIdx.x;
    if (t < 16) pool[0].m[t >> 1][t & 1] = (t & 1) ? 0u : 0xffffffffu;
}

// ---- prune ------------------------------------------------------------------------------
struct PruneArgs {
    const nbx_sci_entry* sci;
    int n_sci, part, nparts;
    const nbx_cj_entry* cj;
    const nbx_mask_pool_entry* pool;
    const float4* xq_i;
    const float4* xq_j;
    float3 box;
    float rli2;
    nbx_sci_entry* sci_in;
    nbx_cj_entry* cj_in;
    int n_cj, n_pool, nsci_i, ncl_j; // list / grid extents (checked builds)
};

constexpr int PRUNE_THREADS = 256;

__global__ void __launch_bounds__(PRUNE_THREADS) k_prune(PruneArgs A)
{
    __shared__ float4 s_xi[PRUNE_THREADS];
    const int lane = threadIdx.x & 31;
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int e = A.part + A.nparts * w;
    if (e >= A.n_sci) return;
    const unsigned lt = (1u << lane) - 1u;
    const nbx_sci_entry se = A.sci[e];
    const float3 v = shift_vec(se.shift, A.box);
    float4* xi = s_xi + (threadIdx.x & ~31);
    {
        const float4 t = A.xq_i[32 * se.sci + lane];
        xi[lane] = make_float4(__fadd_rn(t.x, v.x), __fadd_rn(t.y, v.y), __fadd_rn(t.z, v.z), 0.f);
    }
    __syncwarp();
    int kept = 0;
    for (int c0 = se.cj_start; c0 < se.cj_end; c0 += 32) {
        const int q = c0 + lane;
        nbx_cj_entry my;
        my.cj = 0;
        my.meta = 0u;
        if (q < se.cj_end) my = A.cj[q];
        unsigned nm = 0u;
        const unsigned imask = my.meta & 0xffu, pidx = my.meta >> 8;
        if (imask) {
            float4 xj[8];
#pragma unroll
            for (int j = 0; j < 8; j++) xj[j] = A.xq_j[8 * my.cj + j];
            for (int kk = 0; kk < 8; kk++) {
                if (!(imask & (1u << kk))) continue;
                unsigned pm = 0xffffffffu;
                if (pidx) pm = A.pool[pidx].m[kk][0] | A.pool[pidx].m[kk][1];
                bool hit = false;
                if (pm == 0xffffffffu) {
                    // unmasked tile (the common case): no per-pair mask bits to test
                    for (int i = 0; i < 4 && !hit; i++) {
                        const float4 a = xi[4 * kk + i];
#pragma unroll
                        for (int j = 0; j < 8; j++) {
                            const float dx = __fsub_rn(a.x, xj[j].x);
                            const float dy = __fsub_rn(a.y, xj[j].y);
                            const float dz = __fsub_rn(a.z, xj[j].z);
                            hit |= __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx))) < A.rli2;
                        }
                    }
                } else {
                    for (int i = 0; i < 4 && !hit; i++) {
                        const unsigned row = (pm >> (i * 8)) & 0xffu;
                        if (!row) continue;
                        const float4 a = xi[4 * kk + i];
#pragma unroll
                        for (int j = 0; j < 8; j++) {
                            const float dx = __fsub_rn(a.x, xj[j].x);
                            const float dy = __fsub_rn(a.y, xj[j].y);
                            const float dz = __fsub_rn(a.z, xj[j].z);
                            const float r2 = __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
                            hit |= ((row >> j) & 1u) && (r2 < A.rli2);
                        }
                    }
                }
                if (hit) nm |= 1u << kk;
            }
        }
        const unsigned keep = __ballot_sync(0xffffffffu, nm != 0u);
        if (nm) {
            nbx_cj_entry o;
            o.cj = my.cj;
            o.meta = nm | (my.meta & ~0xffu);
            A.cj_in[se.cj_start + kept + __popc(keep & lt)] = o;
        }
        kept += __popc(keep);
    }
    if (lane == 0) {
        nbx_sci_entry o = se;
        o.cj_end = se.cj_start + kept;
        A.sci_in[e] = o;
    }
}

// Warp-uniform prune: one sci entry per warp, lane = i atom (i-cluster lane/4, row lane%4).
// The 32 cj entries of a chunk are staged in shared memory (8 coalesced 128-B loads), then
// every entry is tested by the whole warp at once: 8 r^2 tests per lane, two ballots give the
// entry's surviving i-cluster bits.  No lane diverges (k_prune's lane-per-entry loop runs
// the worst lane's early exit for all 32), so the warp issues ~8 instructions per lane per
// tested atom pair.  Same r^2 rounding and the same keep rule as k_prune: bit-identical lists.
__global__ void __launch_bounds__(PRUNE_THREADS) k_prune_lanes(PruneArgs A)
{
    __shared__ float4 s_xj[PRUNE_THREADS / 32][32][8];
    const int lane = threadIdx.x & 31;
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int e = A.part + A.nparts * w;
    if (e >= A.n_sci) return;
    const unsigned full = 0xffffffffu, lt = (1u << lane) - 1u;
    const nbx_sci_entry se = A.sci[e];
    const float3 v = shift_vec(se.shift, A.box);
    const float4 t0 = A.xq_i[32 * se.sci + lane];
    const float ax = __fadd_rn(t0.x, v.x), ay = __fadd_rn(t0.y, v.y), az = __fadd_rn(t0.z, v.z);
    const int kk = lane >> 2, ii = lane & 3;
    float4(*xs)[8] = s_xj[threadIdx.x >> 5];
    int kept = 0;
    for (int c0 = se.cj_start; c0 < se.cj_end; c0 += 32) {
        const int cnt = min(32, se.cj_end - c0);
        nbx_cj_entry my;
        my.cj = 0;
        my.meta = 0u;
        if (lane < cnt) my = A.cj[c0 + lane];
        __syncwarp();
        for (int r = 0; r < 8 && 4 * r < cnt; r++) {
            const int t = 4 * r + (lane >> 3);
            const int cjt = __shfl_sync(full, my.cj, t);
            if (t < cnt) xs[t][lane & 7] = A.xq_j[8 * cjt + (lane & 7)];
        }
        __syncwarp();
        unsigned my_nm = 0u;
        for (int t = 0; t < cnt; t++) {
            const unsigned meta = __shfl_sync(full, my.meta, t);
            const unsigned pidx = meta >> 8;
            bool hit = false;
            if (pidx == 0u) {
#pragma unroll
                for (int j = 0; j < 8; j++) {
                    const float4 b = xs[t][j];
                    const float dx = __fsub_rn(ax, b.x);
                    const float dy = __fsub_rn(ay, b.y);
                    const float dz = __fsub_rn(az, b.z);
                    hit |= __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx))) < A.rli2;
                }
            } else {
                const unsigned row = ((A.pool[pidx].m[kk][0] | A.pool[pidx].m[kk][1]) >> (8 * ii)) & 0xffu;
#pragma unroll
                for (int j = 0; j < 8; j++) {
                    const float4 b = xs[t][j];
                    const float dx = __fsub_rn(ax, b.x);
                    const float dy = __fsub_rn(ay, b.y);
                    const float dz = __fsub_rn(az, b.z);
                    const float r2 = __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
                    hit |= ((row >> j) & 1u) && (r2 < A.rli2);
                }
            }
            const unsigned bits = __ballot_sync(full, hit);
            const unsigned nm = __ballot_sync(full, lane < 8 && ((bits >> (4 * (lane & 7))) & 0xfu)) & meta & 0xffu;
            if (lane == t) my_nm = nm;
        }
        const unsigned keep = __ballot_sync(full, my_nm != 0u);
        if (my_nm) {
            nbx_cj_entry o;
            o.cj = my.cj;
            o.meta = my_nm | (my.meta & ~0xffu);
            A.cj_in[se.cj_start + kept + __popc(keep & lt)] = o;
        }
        kept += __popc(keep);
    }
    if (lane == 0) {
        nbx_sci_entry o = se;
        o.cj_end = se.cj_start + kept;
        A.sci_in[e] = o;
    }
}

// Packed prune: the active (cj entry, i-cluster) tiles of a 32-entry chunk -- the outer
// list's imask bits, ~5 of 8 per entry -- are compacted into an item table in shared memory
// and tested 8 tiles per warp pass (4 lanes = the tile's 4 i atoms, 8 j atoms each).  Unlike
// k_prune_lanes it never tests a tile the outer list excluded, and unlike k_prune no lane
// waits on another lane's entry.  The j atoms are staged structure-of-arrays so an unmasked
// pass runs two j atoms per FADD2 / FMUL2 / FFMA2 (the kernel is issue-bound with the FP32
// pipe half idle).  dx = xj - xi is the exact negation of xi - xj, so every r^2 has the
// scalar kernels' rounding and the keep rule is unchanged: bit-identical lists.
// j atoms of a chunk, structure of arrays per coordinate: row t (entry t) = 8 floats at a stride
// of NBX_PRUNE_JS floats.  A pass reads one 16-byte quarter-row (h = 0, 1) of up to 8 distinct
// rows per LDS.128.  With a 12-float stride quarter (t, h) sits in bank quad (3 t + h) mod 8,
// distinct for 8 consecutive t (conflict-free passes, and the staging stores no longer
// conflict); unpadded (8 floats) rows t and t + 4 share a quad.  (Round 1's array-of-rows layout
// x[8] y[8] z[8] at stride 28 put rows t, t + 8 on the same quads and its staging stores 2-way
// conflicted: 171 M conflicts per 12 M-atom prune.)
#ifndef NBX_PRUNE_JS
// 8: rows unpadded (3 KB per warp).  The stride-12 layout above is bank-conflict-free for 8
// consecutive rows but its 4.6 KB per warp costs occupancy: 12 M 3.90 -> 3.82 ms, STMV 0.607 ->
// 0.594 ms with 8 (profiles/r02_prune_variants.jsonl)
#define NBX_PRUNE_JS 8
#endif
#ifndef NBX_PRUNE_MINB
// 6 CTAs/SM (<= 40 registers, no spills; 6 x 33 KB of staging fits the SM's shared memory):
// 12 M prune 3.78 -> 3.49 ms, STMV 0.584 -> 0.555 ms vs the unconstrained 62 registers at 4
// (82k membrane +6 %; profiles/r02_prune_minb.jsonl)
#define NBX_PRUNE_MINB 6
#endif
constexpr int PRUNE_JS = NBX_PRUNE_JS;

#ifndef NBX_PRUNE_REP
// 1: a first sweep tests one row of every active tile (i atom 1 against the 8 j atoms, one lane
// per tile, 32 tiles per warp instruction); only the tiles it does not keep get the full 32-pair
// test.  The row's r^2 are the full test's own (same packed operations), so the kept set and the
// lists are unchanged
#define NBX_PRUNE_REP 1
#endif

// per-warp shared staging of the packed prune
struct PruneWarpSmem {
    float xj[3][32][PRUNE_JS];
    float4 xi[32];
#if !NBX_PRUNE_REP
    unsigned pass[32]; // per pass: the hit ballot (4 lanes per item)
#endif
    unsigned pidx[32];
    unsigned char item[256]; // entry << 3 | i-cluster
#if NBX_PRUNE_REP
    float4 xi1[8];            // row 1 of the 8 i clusters, contiguous: the row sweep's 8
                              // distinct reads hit 8 bank quads (xi's 64-byte stride hits 2)
    unsigned char hit[256];   // per item: kept
    unsigned char item2[256]; // items the row sweep left open (indices into item)
#endif
};

// min r^2 of i atom a against the 8 j atoms of staged row (xs, ys, zs); MASKED: pairs whose bit
// in `row` is clear count as +inf
template <bool MASKED>
__device__ __forceinline__ float prune_r2min8(const float4& a, const float* xs, const float* ys, const float* zs,
                                              unsigned row)
{
    const f2x AX = bc(a.x), AY = bc(a.y), AZ = bc(a.z);
    float r2min = 0.f;
#pragma unroll
    for (int h = 0; h < 2; h++) {
        const ulonglong2 X = *reinterpret_cast<const ulonglong2*>(xs + 4 * h);
        const ulonglong2 Y = *reinterpret_cast<const ulonglong2*>(ys + 4 * h);
        const ulonglong2 Z = *reinterpret_cast<const ulonglong2*>(zs + 4 * h);
        const f2x DX0 = sub2(X.x, AX), DY0 = sub2(Y.x, AY), DZ0 = sub2(Z.x, AZ);
        const f2x DX1 = sub2(X.y, AX), DY1 = sub2(Y.y, AY), DZ1 = sub2(Z.y, AZ);
        const float2 R0 = upk(fma2(DZ0, DZ0, fma2(DY0, DY0, mul2(DX0, DX0))));
        const float2 R1 = upk(fma2(DZ1, DZ1, fma2(DY1, DY1, mul2(DX1, DX1))));
        float m4;
        if (MASKED) {
            const unsigned rb = row >> (4 * h);
            const float inf = __int_as_float(0x7f800000);
            m4 = fminf(fminf((rb & 1u) ? R0.x : inf, (rb & 2u) ? R0.y : inf),
                       fminf((rb & 4u) ? R1.x : inf, (rb & 8u) ? R1.y : inf));
        } else {
            m4 = fminf(fminf(R0.x, R0.y), fminf(R1.x, R1.y));
        }
        r2min = h ? fminf(r2min, m4) : m4;
    }
    return r2min;
}

// one 4-lane-per-tile pass over items it (lane group g = lane / 4, row ii = lane % 4): hit of
// this lane's row.  ROW1: the row sweep (ii == 1, from the contiguous row-1 copy)
template <bool ROW1 = false>
__device__ __forceinline__ bool prune_tile_rows(const PruneArgs& A, const PruneWarpSmem& S, unsigned it, int ii)
{
    const int t = it >> 3, kk = it & 7;
#if NBX_PRUNE_REP
    const float4 a = ROW1 ? S.xi1[kk] : S.xi[4 * kk + ii];
#else
    const float4 a = S.xi[4 * kk + ii];
#endif
    const unsigned pidx = S.pidx[t];
    const float* xs = S.xj[0][t];
    const float* ys = S.xj[1][t];
    const float* zs = S.xj[2][t];
    float r2min;
    if (!__any_sync(0xffffffffu, pidx != 0u)) {
        r2min = prune_r2min8<false>(a, xs, ys, zs, 0xffu);
    } else {
        // a pass holding an excluded (pool) tile: masked pairs' r^2 replaced by +inf
        unsigned row = 0xffu;
        if (pidx) row = ((A.pool[pidx].m[kk][0] | A.pool[pidx].m[kk][1]) >> (8 * ii)) & 0xffu;
        r2min = prune_r2min8<true>(a, xs, ys, zs, row);
    }
    return r2min < A.rli2;
}

// i atoms of sci entry se (+ its shift) into the warp's staging
__device__ __forceinline__ void prune_stage_i(const PruneArgs& A, const nbx_sci_entry& se, PruneWarpSmem& S, int lane)
{
    NBX_DCHECK(se.sci >= 0 && se.sci < A.nsci_i && se.shift >= 0 && se.shift < NBX_NSHIFT && se.cj_start >= 0 &&
               se.cj_end <= A.n_cj);
    const float3 v = shift_vec(se.shift, A.box);
    const float4 t0 = A.xq_i[32 * se.sci + lane];
    const float4 a = make_float4(__fadd_rn(t0.x, v.x), __fadd_rn(t0.y, v.y), __fadd_rn(t0.z, v.z), 0.f);
    S.xi[lane] = a;
#if NBX_PRUNE_REP
    if ((lane & 3) == 1) S.xi1[lane >> 2] = a;
#endif
}

// one chunk of up to 32 cj entries starting at c0 of an entry ending at cj_end: returns this
// lane's entry (my) and its new interaction mask (0: dropped)
__device__ __forceinline__ unsigned prune_chunk_packed(const PruneArgs& A, PruneWarpSmem& S, int lane, int c0,
                                                       int cj_end, nbx_cj_entry& my)
{
    const unsigned full = 0xffffffffu;
    const int g = lane >> 2, ii = lane & 3;
    const int cnt = min(32, cj_end - c0);
    my.cj = 0;
    my.meta = 0u;
    if (lane < cnt) my = A.cj[c0 + lane];
    NBX_DCHECK(lane >= cnt || (my.cj >= 0 && my.cj < A.ncl_j && (int)(my.meta >> 8) < A.n_pool));
    __syncwarp();
    for (int r = 0; r < 8 && 4 * r < cnt; r++) {
        const int t = 4 * r + (lane >> 3);
        const int cjt = __shfl_sync(full, my.cj, t);
        if (t < cnt) {
            const int j = lane & 7;
            const float4 b = A.xq_j[8 * cjt + j];
            S.xj[0][t][j] = b.x;
            S.xj[1][t][j] = b.y;
            S.xj[2][t][j] = b.z;
        }
    }
    // item table: exclusive scan of the entries' active-tile counts
    const unsigned imask = my.meta & 0xffu;
    const int pc = __popc(imask);
    int incl = pc;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int y = __shfl_up_sync(full, incl, d);
        if (lane >= d) incl += y;
    }
    const int total = __shfl_sync(full, incl, 31);
    NBX_DCHECK(total <= 256); // 32 entries x 8 tiles: the item tables' size
    {
        unsigned mm = imask;
        int o = incl - pc;
        while (mm) {
            S.item[o++] = (unsigned char)((lane << 3) | (__ffs(mm) - 1));
            mm &= mm - 1u;
        }
    }
    S.pidx[lane] = my.meta >> 8;
    __syncwarp();
    unsigned my_nm = 0u;
#if NBX_PRUNE_REP
    // sweep 1: one lane per item, row ii = 1 of its tile; the items it does not keep are
    // compacted into item2
    int total2 = 0;
    for (int base = 0; base < total; base += 32) {
        const int m = base + lane;
        const unsigned it = m < total ? S.item[m] : 0u;
        const bool h1 = prune_tile_rows<true>(A, S, it, 1); // every lane: the test holds a warp vote
        const bool hit = m < total && h1;
        if (m < total) S.hit[m] = hit ? 1 : 0;
        const unsigned open = __ballot_sync(full, m < total && !hit);
        if (m < total && !hit) S.item2[total2 + __popc(open & ((1u << lane) - 1u))] = (unsigned char)m;
        total2 += __popc(open);
    }
    __syncwarp();
    // sweep 2: the full 4-row test of the open items, 8 per pass
    for (int base = 0; base < total2; base += 8) {
        const int m2 = base + g;
        const unsigned mi = m2 < total2 ? S.item2[m2] : 0u;
        const unsigned it = S.item[mi];
        const bool hit = prune_tile_rows(A, S, it, ii);
        const unsigned bits = __ballot_sync(full, hit && m2 < total2);
        if (ii == 0 && m2 < total2 && ((bits >> (4 * g)) & 0xfu)) S.hit[mi] = 1;
    }
    __syncwarp();
    // each entry collects its items' hits (items o .. o + pc - 1, in imask bit order)
    {
        unsigned mm = imask;
        for (int m = incl - pc; mm; m++) {
            if (S.hit[m]) my_nm |= mm & (0u - mm);
            mm &= mm - 1u;
        }
    }
#else
    for (int base = 0; base < total; base += 8) {
        const int m = base + g;
        const unsigned it = m < total ? S.item[m] : 0u;
        const bool hit = prune_tile_rows(A, S, it, ii);
        const unsigned bits = __ballot_sync(full, hit && m < total);
        if (lane == 0) S.pass[base >> 3] = bits;
    }
    __syncwarp();
    // each entry collects its items' hits (items o .. o + pc - 1, in imask bit order)
    {
        unsigned mm = imask;
        for (int m = incl - pc; mm; m++) {
            if ((S.pass[m >> 3] >> (4 * (m & 7))) & 0xfu) my_nm |= mm & (0u - mm);
            mm &= mm - 1u;
        }
    }
#endif
    return lane < cnt ? my_nm : 0u;
}

__global__ void __launch_bounds__(PRUNE_THREADS, NBX_PRUNE_MINB) k_prune_packed(PruneArgs A)
{
    constexpr int W = PRUNE_THREADS / 32;
    __shared__ __align__(16) PruneWarpSmem s_w[W];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int e = A.part + A.nparts * w;
    if (e >= A.n_sci) return;
    const unsigned full = 0xffffffffu, lt = (1u << lane) - 1u;
    PruneWarpSmem& S = s_w[wib];
    const nbx_sci_entry se = A.sci[e];
    prune_stage_i(A, se, S, lane);
    int kept = 0;
    for (int c0 = se.cj_start; c0 < se.cj_end; c0 += 32) {
        nbx_cj_entry my;
        const unsigned my_nm = prune_chunk_packed(A, S, lane, c0, se.cj_end, my);
        const unsigned keep = __ballot_sync(full, my_nm != 0u);
        if (my_nm) {
            nbx_cj_entry o;
            o.cj = my.cj;
            o.meta = my_nm | (my.meta & ~0xffu);
            A.cj_in[se.cj_start + kept + __popc(keep & lt)] = o;
        }
        kept += __popc(keep);
        __syncwarp();
    }
    if (lane == 0) {
        nbx_sci_entry o = se;
        o.cj_end = se.cj_start + kept;
        A.sci_in[e] = o;
    }
}

// Split prune for short lists (fewer sci entries than the machine holds warps: small boxes, DD
// halo lists): one warp per (entry, 32-entry chunk) instead of per entry, kept entries
// compacted at the chunk's own offset in a scratch copy, then k_prune_gather moves each entry's
// chunks together -- the same inner list as k_prune_packed, with up to `chunks` x the warps
__global__ void __launch_bounds__(PRUNE_THREADS, NBX_PRUNE_MINB) k_prune_split(PruneArgs A, int chunks,
                                                                                nbx_cj_entry* tmp, int* kept_n)
{
    constexpr int W = PRUNE_THREADS / 32;
    __shared__ __align__(16) PruneWarpSmem s_w[W];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int we = w / chunks, c = w - we * chunks;
    const int e = A.part + A.nparts * we;
    if (e >= A.n_sci) return;
    const unsigned full = 0xffffffffu, lt = (1u << lane) - 1u;
    PruneWarpSmem& S = s_w[wib];
    const nbx_sci_entry se = A.sci[e];
    const int c0 = se.cj_start + 32 * c;
    if (c0 >= se.cj_end) {
        if (lane == 0) kept_n[w] = 0;
        return;
    }
    prune_stage_i(A, se, S, lane);
    nbx_cj_entry my;
    const unsigned my_nm = prune_chunk_packed(A, S, lane, c0, se.cj_end, my);
    const unsigned keep = __ballot_sync(full, my_nm != 0u);
    if (my_nm) {
        nbx_cj_entry o;
        o.cj = my.cj;
        o.meta = my_nm | (my.meta & ~0xffu);
        NBX_DCHECK(c0 + __popc(keep & lt) < A.n_cj);
        tmp[c0 + __popc(keep & lt)] = o;
    }
    if (lane == 0) kept_n[w] = __popc(keep);
}

__global__ void __launch_bounds__(256) k_prune_gather(PruneArgs A, int chunks, const nbx_cj_entry* __restrict__ tmp,
                                                      const int* __restrict__ kept_n)
{
    const int lane = threadIdx.x & 31;
    const int we = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int e = A.part + A.nparts * we;
    if (e >= A.n_sci) return;
    const nbx_sci_entry se = A.sci[e];
    int kept = 0;
    for (int c = 0; c < chunks; c++) {
        const int n = kept_n[we * chunks + c];
        if (lane < n) A.cj_in[se.cj_start + kept + lane] = tmp[se.cj_start + 32 * c + lane];
        kept += n;
    }
    if (lane == 0) {
        nbx_sci_entry o = se;
        o.cj_end = se.cj_start + kept;
        A.sci_in[e] = o;
    }
}

// Fixed-lane prune (NBX_PRUNE_KERNEL=3): lane = i atom of the super-cluster (i-cluster lane / 4,
// row lane % 4), its shifted coordinates in registers for the whole entry; the chunk's j atoms
// staged structure-of-arrays (row t = 8 floats: the staging stores hit 32 consecutive words,
// every read is a broadcast of one row).  Each cj entry is one warp-uniform pass: every lane
// tests its i atom against the 8 j atoms with packed FP32x2 r^2 (two j atoms per FADD2 /
// FMUL2 / FFMA2), one ballot, and the 32 hit bits fold into the entry's 8 i-cluster bits.
// No item table, no shared atomics; inactive tiles (imask bit clear) are computed and
// discarded, so it trades ~3/8 wasted lanes for the packed kernel's bookkeeping.  Same r^2
// rounding (dx = xj - xi, the exact negation) and keep rule: bit-identical lists.
__global__ void __launch_bounds__(PRUNE_THREADS) k_prune_fixed(PruneArgs A)
{
    constexpr int W = PRUNE_THREADS / 32;
    __shared__ __align__(16) float s_j[W][3][32][8];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int e = A.part + A.nparts * w;
    if (e >= A.n_sci) return;
    const unsigned full = 0xffffffffu, lt = (1u << lane) - 1u;
    const nbx_sci_entry se = A.sci[e];
    const int kk = lane >> 2, ii = lane & 3;
    f2x AX, AY, AZ;
    {
        const float3 v = shift_vec(se.shift, A.box);
        const float4 t0 = A.xq_i[32 * se.sci + lane];
        AX = bc(__fadd_rn(t0.x, v.x));
        AY = bc(__fadd_rn(t0.y, v.y));
        AZ = bc(__fadd_rn(t0.z, v.z));
    }
    int kept = 0;
    for (int c0 = se.cj_start; c0 < se.cj_end; c0 += 32) {
        const int cnt = min(32, se.cj_end - c0);
        nbx_cj_entry my;
        my.cj = 0;
        my.meta = 0u;
        if (lane < cnt) my = A.cj[c0 + lane];
        __syncwarp();
        for (int r = 0; r < 8 && 4 * r < cnt; r++) {
            const int t = 4 * r + (lane >> 3);
            const int cjt = __shfl_sync(full, my.cj, t);
            if (t < cnt) {
                const int j = lane & 7;
                const float4 b = A.xq_j[8 * cjt + j];
                s_j[wib][0][t][j] = b.x;
                s_j[wib][1][t][j] = b.y;
                s_j[wib][2][t][j] = b.z;
            }
        }
        __syncwarp();
        unsigned my_nm = 0u;
        for (int t = 0; t < cnt; t++) {
            const unsigned meta = __shfl_sync(full, my.meta, t);
            const unsigned pidx = meta >> 8;
            const float* xs = s_j[wib][0][t];
            const float* ys = s_j[wib][1][t];
            const float* zs = s_j[wib][2][t];
            float R[8];
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const ulonglong2 X = *reinterpret_cast<const ulonglong2*>(xs + 4 * h);
                const ulonglong2 Y = *reinterpret_cast<const ulonglong2*>(ys + 4 * h);
                const ulonglong2 Z = *reinterpret_cast<const ulonglong2*>(zs + 4 * h);
                const f2x DX0 = sub2(X.x, AX), DY0 = sub2(Y.x, AY), DZ0 = sub2(Z.x, AZ);
                const f2x DX1 = sub2(X.y, AX), DY1 = sub2(Y.y, AY), DZ1 = sub2(Z.y, AZ);
                const float2 R0 = upk(fma2(DZ0, DZ0, fma2(DY0, DY0, mul2(DX0, DX0))));
                const float2 R1 = upk(fma2(DZ1, DZ1, fma2(DY1, DY1, mul2(DX1, DX1))));
                R[4 * h] = R0.x;
                R[4 * h + 1] = R0.y;
                R[4 * h + 2] = R1.x;
                R[4 * h + 3] = R1.y;
            }
            if (pidx) { // warp-uniform: the entry holds an excluded pair; masked pairs never keep a tile
                const unsigned row = ((A.pool[pidx].m[kk][0] | A.pool[pidx].m[kk][1]) >> (8 * ii)) & 0xffu;
                const float inf = __int_as_float(0x7f800000);
#pragma unroll
                for (int q = 0; q < 8; q++) R[q] = ((row >> q) & 1u) ? R[q] : inf;
            }
            const float r2min = fminf(fminf(fminf(R[0], R[1]), fminf(R[2], R[3])),
                                      fminf(fminf(R[4], R[5]), fminf(R[6], R[7])));
            const unsigned bits = __ballot_sync(full, r2min < A.rli2);
            // bit 4k of f = OR of bits 4k..4k+3 (i-cluster k hit), gathered into bit k
            unsigned f = bits | (bits >> 1);
            f = (f | (f >> 2)) & 0x11111111u;
            f = (f | (f >> 3)) & 0x03030303u;
            f = (f | (f >> 6)) & 0x000f000fu;
            f = (f | (f >> 12)) & 0xffu;
            if (lane == t) my_nm = f & meta & 0xffu;
        }
        const unsigned keep = __ballot_sync(full, my_nm != 0u);
        if (my_nm) {
            nbx_cj_entry o;
            o.cj = my.cj;
            o.meta = my_nm | (my.meta & ~0xffu);
            A.cj_in[se.cj_start + kept + __popc(keep & lt)] = o;
        }
        kept += __popc(keep);
        __syncwarp();
    }
    if (lane == 0) {
        nbx_sci_entry o = se;
        o.cj_end = se.cj_start + kept;
        A.sci_in[e] = o;
    }
}

// count interacting in-cut-off pairs and pair slots of the inner list (bench denominator)
__global__ void __launch_bounds__(256) k_count_pairs(PruneArgs A, float rc2, unsigned long long* out)
{
    const int lane = threadIdx.x & 31;
    const int e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (e >= A.n_sci) return;
    const nbx_sci_entry se = A.sci_in[e];
    const float3 v = shift_vec(se.shift, A.box);
    const int i = lane >> 3, j = lane & 7;
    unsigned long long np = 0, ns = 0;
    for (int c = se.cj_start; c < se.cj_end; c++) {
        const nbx_cj_entry ce = A.cj_in[c];
        const unsigned imask = ce.meta & 0xffu, pidx = ce.meta >> 8;
        const float4 xj = A.xq_j[8 * ce.cj + j];
        for (int kk = 0; kk < 8; kk++) {
            if (!(imask & (1u << kk))) continue;
            const unsigned im = pidx ? A.pool[pidx].m[kk][0] : 0xffffffffu;
            const float4 t = A.xq_i[32 * se.sci + 4 * kk + i];
            const float dx = __fsub_rn(__fadd_rn(t.x, v.x), xj.x);
            const float dy = __fsub_rn(__fadd_rn(t.y, v.y), xj.y);
            const float dz = __fsub_rn(__fadd_rn(t.z, v.z), xj.z);
            const float r2 = __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
            np += (((im >> lane) & 1u) && r2 < rc2) ? 1 : 0;
            ns += 1;
        }
    }
    for (int o = 16; o > 0; o >>= 1) np += __shfl_xor_sync(0xffffffffu, np, o);
    if (lane == 0) {
        atomicAdd(&out[0], np);
        atomicAdd(&out[1], ns);
    }
}

static PruneArgs prune_args(nbx_ctx* ctx, List& L)
{
    PruneArgs A;
    A.sci = L.sci.p;
    A.n_sci = (int)L.n_sci;
    A.part = 0;
    A.nparts = 1;
    A.cj = L.cj.p;
    A.pool = L.pool.p;
    A.xq_i = ctx->grid[L.gi].xq.p;
    A.xq_j = ctx->grid[L.gj].xq.p;
    A.box = make_float3(ctx->box[0], ctx->box[1], ctx->box[2]);
    A.rli2 = ctx->c.rli2;
    A.sci_in = L.sci_in.p;
    A.cj_in = L.cj_in.p;
    A.n_cj = (int)L.n_cj;
    A.n_pool = (int)L.n_pool;
    A.nsci_i = ctx->grid[L.gi].nsci;
    A.ncl_j = ctx->grid[L.gj].nslots / 8;
    return A;
}

void count_pairs(nbx_ctx* ctx, int l, long long* pairs, long long* slots, cudaStream_t st)
{
    List& L = ctx->list[l];
    if (!L.built) throw CudaError{cudaErrorInvalidValue, "count before search"};
    *pairs = 0;
    *slots = 0;
    if (L.n_sci == 0) return;
    PruneArgs A = prune_args(ctx, L);
    DBuf<unsigned long long>& out = L.pair_count;
    out.ensure(2);
    NBX_CUDA(cudaMemsetAsync(out.p, 0, 2 * sizeof(unsigned long long), st));
    k_count_pairs<<<(int)((L.n_sci * 32 + 255) / 256), 256, 0, st>>>(A, ctx->c.rc2, out.p);
    ctx->launches++;
    NBX_CUDA(cudaGetLastError());
    unsigned long long h[2];
    NBX_CUDA(cudaMemcpyAsync(h, out.p, sizeof(h), cudaMemcpyDeviceToHost, st));
    NBX_CUDA(cudaStreamSynchronize(st));
    *pairs = (long long)h[0];
    *slots = 32ll * (long long)h[1];
}

// Row f2 (the paper's post-prune list sort): order the
// inner list's sci entries longest first, so the persistent force kernel's dynamic
// scheduler starts the long entries early and the tail is short.  Stable radix sort on the
// inverted length: deterministic.
__global__ void k_entry_len(const nbx_sci_entry* __restrict__ sci, int n, unsigned* __restrict__ key,
                            int* __restrict__ idx)
{
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n) return;
    key[e] = 0xffffffffu - (unsigned)(sci[e].cj_end - sci[e].cj_start);
    idx[e] = e;
}

// resident force-kernel warps: 3 CTAs x 8 warps per SM (force.cu FORCE_MIN_BLOCKS x threads / 32)
static bool entry_order_on(const nbx_ctx* ctx, const List& L)
{
    if (ctx->entry_order >= 0) return ctx->entry_order != 0;
    // tabulated Ewald: the sorted order measured slower (STMV flavour +2.9 %, Grappa +0.3 % with
    // the sort's cost on prune steps; profiles/r02_entry_order*.jsonl)
    if (ctx->p.coulomb_type == NBX_COULOMB_EWALD_TAB) return false;
    const int64_t warps = (int64_t)ctx->num_sms * 3 * 8;
    return L.n_sci >= 1024 && L.n_sci < 32 * warps;
}

static void sort_entries(nbx_ctx* ctx, List& L, cudaStream_t st)
{
    const int n = (int)L.n_sci;
    if (n == 0) return;
    L.len_key.ensure(n); L.len_key_out.ensure(n); L.order_in.ensure(n); L.order.ensure(n);
    k_entry_len<<<(n + 255) / 256, 256, 0, st>>>(L.sci_in.p, n, L.len_key.p, L.order_in.p);
    ctx->launches++;
    NBX_CUDA(cudaGetLastError());
    size_t tb = 0;
    NBX_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, L.len_key.p, L.len_key_out.p, L.order_in.p,
                                             L.order.p, n, 0, 32, st));
    L.sort_tmp.ensure(tb + 16);
    NBX_CUDA(cub::DeviceRadixSort::SortPairs(L.sort_tmp.p, tb, L.len_key.p, L.len_key_out.p, L.order_in.p,
                                             L.order.p, n, 0, 32, st));
    ctx->launches += 4;
}

// split prune when the entries to prune fill less than half a wave of prune warps (16 of the
// 32 per SM): there the per-entry warps are latency-bound and the chunks give the SMs more
// warps (water 3k 24.6 -> 19.8 us, RNase 24k 53.4 -> 47.7 us); from about a wave on, the
// chunks' repeated i staging and the gather pass cost more (82k membrane 70 -> 88 us, STMV
// 0.58 -> 0.89 ms forced on; profiles/r02_prune_split.jsonl)
static bool prune_split_on(const nbx_ctx* ctx, int nw)
{
    if (ctx->prune_split >= 0) return ctx->prune_split > 0;
    return nw < 16 * ctx->num_sms;
}

void prune(nbx_ctx* ctx, int l, int part, int nparts, cudaStream_t st)
{
    List& L = ctx->list[l];
    if (!L.built) throw CudaError{cudaErrorInvalidValue, "prune before search"};
    if (L.n_sci == 0) return;
    PruneArgs A = prune_args(ctx, L);
    A.part = part;
    A.nparts = nparts;
    const int nw = (int)((L.n_sci - part + nparts - 1) / nparts);
    if (nw <= 0) return;
    const int blocks = (nw * 32 + PRUNE_THREADS - 1) / PRUNE_THREADS;
    if (ctx->prune_kernel == 2 && L.prune_chunks >= 2 && prune_split_on(ctx, nw)) {
        const int chunks = L.prune_chunks;
        k_prune_split<<<(int)(((long long)nw * chunks * 32 + PRUNE_THREADS - 1) / PRUNE_THREADS), PRUNE_THREADS, 0, st>>>(
            A, chunks, L.prune_tmp.p, L.prune_kept.p);
        k_prune_gather<<<(nw * 32 + 255) / 256, 256, 0, st>>>(A, chunks, L.prune_tmp.p, L.prune_kept.p);
        ctx->launches += 2;
    } else if (ctx->prune_kernel == 0) k_prune<<<blocks, PRUNE_THREADS, 0, st>>>(A);
    else if (ctx->prune_kernel == 1) k_prune_lanes<<<blocks, PRUNE_THREADS, 0, st>>>(A);
    else if (ctx->prune_kernel == 3) k_prune_fixed<<<blocks, PRUNE_THREADS, 0, st>>>(A);
    else k_prune_packed<<<blocks, PRUNE_THREADS, 0, st>>>(A); // default
    ctx->launches++;
    NBX_CUDA(cudaGetLastError());
    L.use_order = entry_order_on(ctx, L);
    if (L.use_order) sort_entries(ctx, L, st);
}

// search in two halves around the host read of the list sizes (search_begin: kernels, scans
// and an async read into pinned memory; search_end, after the caller's wait: allocation,
// compaction or fill, prune), so search_pair can overlap the local and nonlocal lists
struct SearchStage {
    SearchArgs A;
    bool single = false;
    int blocks = 0, nsci = 0;
    int* h = nullptr; // pinned: [0..2] entry / cj / pool totals, [3..6] flags
};

static void search_begin(nbx_ctx* ctx, int l, cudaStream_t st, SearchStage& S)
{
    List& L = ctx->list[l];
    L.mode = l;
    L.gi = 0;
    L.gj = (l == NBX_LIST_LOCAL) ? 0 : 1;
    Grid& GI = ctx->grid[L.gi];
    Grid& GJ = ctx->grid[L.gj];
    if (!GI.built || !GJ.built) throw CudaError{cudaErrorInvalidValue, "search before grid build"};
    const int nsci = GI.nsci;
    SearchArgs A;
    A.bb_ci = GI.bb_ci.p;
    A.bb_sci = GI.bb_sci.p;
    A.order_i = GI.order.p;
    A.gid_i = GI.gid.p;
    A.nsci_i = nsci;
    A.bb_cj = GJ.bb_cj.p;
    A.bb_sci_j = GJ.bb_sci.p;
    A.order_j = GJ.order.p;
    A.gid_j = GJ.gid.p;
    A.slotmap_j = GJ.slotmap.p;
    A.col_start_j = GJ.col_start.p;
    A.bb_col_j = GJ.bb_col.p;
    A.ncx_j = GJ.ncx;
    A.ncy_j = GJ.ncy;
    A.lo_jx = GJ.lo[0];
    A.lo_jy = GJ.lo[1];
    A.inv_jx = GJ.inv_cell[0];
    A.inv_jy = GJ.inv_cell[1];
    A.excl_off = ctx->excl_off_g.p;
    A.excl_gid = ctx->excl_gid_g.p;
    A.box = make_float3(ctx->box[0], ctx->box[1], ctx->box[2]);
    A.pbc0 = ctx->pbc[0];
    A.pbc1 = ctx->pbc[1];
    A.pbc2 = ctx->pbc[2];
    A.mode = L.mode;
    A.rl = ctx->p.rlist_outer;
    A.rl2 = ctx->c.rlo2;
    A.rlm = ctx->p.rlist_outer * 1.001f + 1.0e-4f;
    A.ncl_j = GJ.nslots / 8;

    const int n3 = 3 * (nsci + 1);
    L.counts.ensure(n3);
    L.offsets.ensure(n3);
    L.flags.ensure(4);
    NBX_CUDA(cudaMemsetAsync(L.counts.p, 0, sizeof(int) * n3, st));
    NBX_CUDA(cudaMemsetAsync(L.flags.p, 0, sizeof(int) * 4, st));
    A.counts = L.counts.p;
    A.offsets = L.offsets.p;
    A.flags = L.flags.p;
    const int blocks = (nsci * 32 + SEARCH_THREADS - 1) / SEARCH_THREADS;
    // Single pass when a previous search sized the per-sci capacities (the list structure
    // changes little between searches); otherwise, or on overflow, count + fill.
    const bool single = L.cap_cj > 0 && nsci > 0;
    if (single) {
        L.tsci.ensure((size_t)NBX_NSHIFT * nsci);
        L.tcj.ensure((size_t)L.cap_cj * nsci);
        L.tpool.ensure((size_t)L.cap_pool * nsci);
        A.cap_cj = L.cap_cj;
        A.cap_pool = L.cap_pool;
        A.sci_out = L.tsci.p;
        A.cj_out = L.tcj.p;
        A.pool_out = L.tpool.p;
        k_search<SEARCH_SINGLE><<<blocks, SEARCH_THREADS, 0, st>>>(A);
        ctx->launches++;
        NBX_CUDA(cudaGetLastError());
    } else if (nsci > 0) {
        k_search<SEARCH_COUNT><<<blocks, SEARCH_THREADS, 0, st>>>(A);
        ctx->launches++;
        NBX_CUDA(cudaGetLastError());
    }
    size_t tb = 0;
    NBX_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, L.counts.p, L.offsets.p, nsci + 1, st));
    L.tmp.ensure(tb + 16);
    for (int k = 0; k < 3; k++) {
        NBX_CUDA(cub::DeviceScan::ExclusiveSum(L.tmp.p, tb, L.counts.p + k * (nsci + 1),
                                               L.offsets.p + k * (nsci + 1), nsci + 1, st));
        ctx->launches++;
    }
    S.A = A;
    S.single = single;
    S.blocks = blocks;
    S.nsci = nsci;
    S.h = host_pin(ctx) + 8 + 8 * l;
    for (int k = 0; k < 3; k++)
        NBX_CUDA(cudaMemcpyAsync(S.h + k, L.offsets.p + k * (nsci + 1) + nsci, sizeof(int),
                                 cudaMemcpyDeviceToHost, st));
    NBX_CUDA(cudaMemcpyAsync(S.h + 3, L.flags.p, 4 * sizeof(int), cudaMemcpyDeviceToHost, st));
}

static void search_end(nbx_ctx* ctx, int l, cudaStream_t st, SearchStage& S)
{
    List& L = ctx->list[l];
    SearchArgs& A = S.A;
    const bool single = S.single;
    const int blocks = S.blocks, nsci = S.nsci;
    const int* tot = S.h;
    const int* fl = S.h + 3;
    L.n_sci = tot[0];
    L.n_cj = tot[1];
    L.n_pool = (int64_t)tot[2] + 1;
    if (L.n_pool >= (1ll << 24)) throw CudaError{cudaErrorMemoryAllocation, "mask pool exceeds 24-bit index"};
    L.sci.ensure(L.n_sci + 1);
    L.sci_in.ensure(L.n_sci + 1);
    L.cj.ensure(L.n_cj + 1);
    L.cj_in.ensure(L.n_cj + 1);
    L.pool.ensure(L.n_pool);
    k_pool0<<<1, 32, 0, st>>>(L.pool.p);
    ctx->launches++;
    if (single && !fl[0]) {
        k_compact<<<blocks, SEARCH_THREADS, 0, st>>>(nsci, L.counts.p, L.offsets.p, L.cap_cj, L.cap_pool, L.tsci.p,
                                                     L.tcj.p, L.tpool.p, L.sci.p, L.cj.p, L.pool.p);
        ctx->launches++;
        NBX_CUDA(cudaGetLastError());
    } else if (nsci > 0) {
        A.sci_out = L.sci.p;
        A.cj_out = L.cj.p;
        A.pool_out = L.pool.p;
        k_search<SEARCH_FILL><<<blocks, SEARCH_THREADS, 0, st>>>(A);
        ctx->launches++;
        NBX_CUDA(cudaGetLastError());
    }
    // capacities for the next single pass: 50 % headroom over this search's maxima.  The private
    // buffers (nsci x cap) are reallocated outside the next search; a regrow is a multi-GB
    // cudaFree + cudaMalloc (tens of ms, and it contends with NVML polls for the driver lock).
    // Regrown only after a search that did not fit (fl[0]: it fell back to count + fill, which
    // needs no private buffers), or on the first: a regrow inside an MD run is a rare event tied
    // to a search that was slow anyway (round 2: regrowing whenever 25 % headroom was lost cost
    // a multi-GB reallocation every few hundred steps on some DD ranks)
    if (L.cap_cj == 0 || fl[0]) {
        const int ncap = fl[1] + fl[1] / 2 + 32, pcap = fl[2] + fl[2] / 2 + 8;
        if (ncap > L.cap_cj) L.cap_cj = ncap;
        if (pcap > L.cap_pool) L.cap_pool = pcap;
    }
    if (nsci > 0) {
        L.tsci.ensure((size_t)NBX_NSHIFT * nsci);
        L.tcj.ensure((size_t)L.cap_cj * nsci);
        L.tpool.ensure((size_t)L.cap_pool * nsci);
    }
    // split-prune scratch (sized here, never inside a step): chunks of the longest sci's
    // entries; an entry is at most one sci's cj entries (fl[1] is the largest of those)
    L.prune_chunks = 0;
    if (ctx->prune_kernel == 2 && L.n_sci > 0 && prune_split_on(ctx, (int)L.n_sci)) {
        const int chunks = (fl[1] + 31) / 32;
        if (chunks >= 2) {
            L.prune_tmp.ensure(L.n_cj + 1);
            L.prune_kept.ensure((size_t)L.n_sci * chunks);
            L.prune_chunks = chunks;
        }
    }
    L.built = true;
    prune(ctx, l, 0, 1, st);
}

void search(nbx_ctx* ctx, int l, cudaStream_t st)
{
    SearchStage S;
    search_begin(ctx, l, st, S);
    NBX_CUDA(cudaStreamSynchronize(st));
    search_end(ctx, l, st, S);
}

void search_pair(nbx_ctx* ctx, cudaStream_t st0, cudaStream_t st1)
{
    SearchStage S0, S1;
    search_begin(ctx, 0, st0, S0);
    search_begin(ctx, 1, st1, S1);
    NBX_CUDA(cudaStreamSynchronize(st0));
    NBX_CUDA(cudaStreamSynchronize(st1));
    search_end(ctx, 0, st0, S0);
    search_end(ctx, 1, st1, S1);
}

} // namespace nbx
