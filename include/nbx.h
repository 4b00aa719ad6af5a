/*
 * nbx.h -- C-ABI of the B200-native NBNXM cluster-pair nonbonded engine (libnbx.so).
 *
 * The reference (arxiv/paper_2405_01420 = the `mdgpusim` step-schedule simulator) has no
 * physics API: its whole representation of this hot path is the cost law
 *     CostTable.duration_ns(kind, atoms, backend, scale)      pkg/src/mdgpusim/costs.py:137-140
 * priced per KernelKind (costs.py:28-43) and submitted per MD step by pipeline.simulate
 * (pipeline.py:222-261 single rank, 321-431 domain-decomposed).  Each entry point below is
 * the real computation behind one of those simulated kernels; the replaced reference
 * interface is cited on each declaration.  DESIGN.md pins the physics, the cluster
 * geometry and the list format that the reference leaves unspecified.
 *
 * Conventions
 *  - Plain C types only.  "dev" pointers are CUDA device pointers on the context's device,
 *    "host" pointers are host memory.  Streams are cudaStream_t passed as void*.
 *  - Every function returns an nbx_status; on failure nbx_last_error() returns a
 *    thread-local message.  No C++ exception crosses the ABI.
 *  - One context = one device; calls on one context are stream-ordered and NOT thread-safe.
 *  - There is no CPU fallback: without a usable sm_100 device nbx_create fails with
 *    NBX_ECUDA.
 *
 * Units: nm, ps, e, kJ/mol.  Coordinates/forces are float32 [n][3].
 */
#ifndef NBX_H
#define NBX_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NBX_API __attribute__((visibility("default")))

/* ---- status codes ---------------------------------------------------------------------- */
typedef enum {
    NBX_OK = 0,
    NBX_EINVAL = 1,         /* bad argument / call order                                   */
    NBX_ECUDA = 2,          /* CUDA runtime error or no sm_100 device                      */
    NBX_ENOMEM = 3,         /* device allocation failed                                    */
    NBX_ELIST_OVERFLOW = 4, /* list or mask pool larger than the 24-bit pool index allows  */
    NBX_ENCCL = 5           /* reserved for the halo layer                                 */
} nbx_status;

/* ---- parameters (mirrors the reference's per-system knobs, presets.py:28-49) ------------ */
/* EWALD_TAB: Ewald real space with the long-range correction force (and, in energy kernels,
 * potential) linearly interpolated from a uniform table in r instead of the fitted rational:
 * the paper's kernel flavour for both its benchmarks. */
enum { NBX_COULOMB_RF = 0, NBX_COULOMB_EWALD = 1, NBX_COULOMB_EWALD_TAB = 2 };
/* LJ modifiers: potential shift (default) or force switch between rvdw_switch and rc
 * (the CHARMM/STMV flavour of the paper).
 * COMB_GEOM / COMB_LB: potential-shifted LJ with a combination rule -- the "Lennard-Jones
 * with combination rule" kernel flavour of the paper's Grappa benchmarks.
 * Pair parameters come from per-type parameters derived (in double, rounded once) from the
 * table's diagonal instead of from the type-pair table:
 *   GEOM: p_t = (sqrt(6 c6_tt), sqrt(12 c12_tt));   6 c6_ij = p6_i p6_j, 12 c12_ij = p12_i p12_j
 *   LB:   sigma_t^6 = c12_tt / c6_tt, eps_t = c6_tt^2 / (4 c12_tt) (0, 0 for c6_tt = 0);
 *         p_t = (sigma_t / 2, sqrt(24 eps_t));  s = s_i + s_j, s6 = ((s s)(s s))(s s),
 *         6 c6_ij = (e_i e_j) s6, 12 c12_ij = 2 ((6 c6_ij) s6)
 * nbx_set_topology checks that every off-diagonal table entry follows the rule (relative
 * 1e-4) and fails with NBX_EINVAL otherwise.                                              */
enum { NBX_LJ_POT_SHIFT = 0, NBX_LJ_FORCE_SWITCH = 1, NBX_LJ_COMB_GEOM = 2, NBX_LJ_COMB_LB = 3 };

typedef struct nbx_params {
    int32_t coulomb_type; /* NBX_COULOMB_RF, NBX_COULOMB_EWALD or NBX_COULOMB_EWALD_TAB     */
    float rc;             /* common LJ/Coulomb cut-off (presets.py:40 cutoff_nm)           */
    float rlist_outer;    /* pair-search radius, list lifetime nstlist (presets.py:44)     */
    float rlist_inner;    /* dynamic-prune radius, lifetime prune_every (presets.py:45)    */
    float epsilon_r;      /* relative dielectric constant                                  */
    float epsilon_rf;     /* reaction-field dielectric; 0 means infinity                   */
    float ewald_rtol;     /* erfc(beta*rc) = ewald_rtol                                    */
    int32_t lj_modifier;  /* NBX_LJ_POT_SHIFT, NBX_LJ_FORCE_SWITCH, NBX_LJ_COMB_GEOM, _LB     */
    float rvdw_switch;    /* force-switch start r1, 0 <= r1 < rc (ignored for POT_SHIFT)   */
} nbx_params;

/* Derived constants, computed identically (double, then rounded once) by the library and
 * by the CPU oracle; exported so tests can check them.                                    */
typedef struct nbx_consts {
    float epsfac;   /* 138.935458 / epsilon_r                                            */
    float k_rf;     /* RF: (eps_rf-eps_r)/((2eps_rf+eps_r) rc^3), or 1/(2rc^3) if eps_rf=inf */
    float c_rf;     /* RF: 1/rc + k_rf rc^2                                               */
    float beta;     /* Ewald splitting coefficient (1/nm)                                 */
    float sh_ewald; /* erfc(beta rc)/rc                                                   */
    float sh_lj6;   /* rc^-6                                                              */
    float sh_lj12;  /* rc^-12                                                             */
    float rc2;      /* rc^2                                                               */
    float rlo2;     /* rlist_outer^2                                                      */
    float rli2;     /* rlist_inner^2                                                      */
    /* force switch: F_a(r) = a r^-(a+1) + A_a (r-r1)^2 + B_a (r-r1)^3 for r1 <= r < rc,
     * V_a(r) = r^-a - A_a/3 (r-r1)^3 - B_a/4 (r-r1)^4 - C_a  (a = 6, 12; GROMACS convention) */
    float fsw_r1;
    float fsw_a6, fsw_b6, fsw_a12, fsw_b12;   /* A_a / a, B_a / a  (tables hold a * c_a)     */
    float fsw_p6, fsw_q6, fsw_p12, fsw_q12;   /* A_a / 3, B_a / 4                            */
    float fsw_c6, fsw_c12;                    /* C_a                                          */
    /* EWALD_TAB: nodes r_k = k / tab_scale, k < tab_n; tab_scale = max(400 beta, 600) /nm,
     * tab_n = ceil(rc tab_scale) + 2.  Force table F_k = beta^3 G(beta^2 r_k^2) (the
     * correction in F/r = qq (r^-3 - F(r))), potential table V_k = erf(beta r_k) / r_k, each
     * stored as (value, next - value) pairs (nbx_ewald_table).                             */
    float tab_scale;
    int32_t tab_n;
} nbx_consts;

/* ---- pair-list format ----------------------------------------
 * Cluster geometry: i-cluster = 4 atoms, j-cluster = 8 atoms = i-clusters {2cj, 2cj+1},
 * super-cluster (sci) = 32 atoms = i-clusters 8sci..8sci+7 = j-clusters 4sci..4sci+3.
 * A list is: sci entries (sci, shift, [cj_start, cj_end)), cj entries (cj, imask | pool<<8)
 * and a mask pool; pool[0] is implicit "all pairs interact, no exclusion correction".   */
typedef struct nbx_sci_entry {
    int32_t sci;
    int32_t shift;    /* 0..26 = (sz+1)*9 + (sy+1)*3 + (sx+1); 13 is the central image */
    int32_t cj_start;
    int32_t cj_end;
} nbx_sci_entry;

typedef struct nbx_cj_entry {
    int32_t cj;
    uint32_t meta; /* bits 0-7: i-cluster interaction mask, bits 8-31: mask-pool index    */
} nbx_cj_entry;

/* pool element p: 8 i-clusters x {interaction mask, exclusion-correction mask}, each a
 * 32-bit word with bit (i*8 + j) for i-atom i (0..3) and j-atom j (0..7).                */
typedef struct nbx_mask_pool_entry {
    uint32_t m[8][2];
} nbx_mask_pool_entry;

enum { NBX_NSHIFT = 27, NBX_CENTRAL_SHIFT = 13 };
enum { NBX_LIST_LOCAL = 0, NBX_LIST_NONLOCAL = 1 };
enum { NBX_GRID_LOCAL = 0, NBX_GRID_NONLOCAL = 1 };

/* force flags */
enum {
    NBX_FORCE_ENERGY = 1u << 0, /* accumulate E_lj, E_coul (fp64)                         */
    NBX_FORCE_VIRIAL = 1u << 1  /* accumulate shift forces for the virial                 */
};

typedef struct nbx_ctx nbx_ctx;

/* ---- lifecycle ------------------------------------------------------------------------- */
NBX_API const char* nbx_last_error(void);
NBX_API const char* nbx_version(void);

/* Derive the constants of a parameter set (no device needed).                           */
NBX_API int nbx_derive_consts(const nbx_params* p, nbx_consts* out);
/* EWALD_TAB tables for derived constants c: ftab[2 * tab_n] and vtab[2 * tab_n] (host). */
NBX_API int nbx_ewald_table(const nbx_consts* c, float* ftab, float* vtab);

/* Create a context on `device` (must be sm_100).  Replaces the reference's per-rank device
 * construction (_RankBuild -> Device/RankRuntime, runtime.py:255-304).                   */
NBX_API int nbx_create(int device, const nbx_params* p, nbx_ctx** out);
NBX_API int nbx_destroy(nbx_ctx* ctx);

/* Topology over the GLOBAL atom set (host arrays; uploaded once).
 * q[n], type[n] in [0,ntypes), c6c12[ntypes*ntypes*2] = plain (c6, c12) with
 * V = c12/r^12 - c6/r^6, exclusions CSR over global ids (symmetric, self not listed).
 * Replaces the per-system sizes of SystemPreset (presets.py:28-60).                      */
NBX_API int nbx_set_topology(nbx_ctx* ctx, int32_t natoms_global, const float* q_host,
                             const int32_t* type_host, int32_t ntypes,
                             const float* c6c12_host, const int32_t* excl_offsets_host,
                             const int32_t* excl_gids_host);

/* Rectangular box edges (nm) and per-dimension periodicity of the searched images
 * (0 for dimensions split by domain decomposition, whose images arrive as halo atoms).    */
NBX_API int nbx_set_box(nbx_ctx* ctx, const float box_host[3], const int32_t pbc_host[3]);

/* ---- grid + pair search: KernelKind.PAIR_SEARCH (costs.py:32,163; pipeline.py:226-230)
 * Build grid `grid` from n atoms: x_dev[n][3] (user order), gid_dev[n] global ids
 * (NULL = identity, single domain).  Region [lo, lo+size) in nm (single domain: 0, box). */
NBX_API int nbx_grid_build(nbx_ctx* ctx, int grid, int32_t n, const float* x_dev,
                           const int32_t* gid_dev, const float lo_host[3],
                           const float size_host[3], void* stream);

/* Build list `list` (LOCAL: grid0 x grid0 half list; NONLOCAL: every grid0 i x grid1 j pair,
 * grid 1 holding a half-shell halo) at rlist_outer, then prune it to
 * rlist_inner.  Synchronises `stream`
 * once to size the list (count pass -> exact allocation -> fill pass).                   */
NBX_API int nbx_search(nbx_ctx* ctx, int list, void* stream);

/* ---- the DD search step's grid builds and searches, overlapped (pipeline.py:329-334, the
 * decomposed step's pair_search on the home atoms + the nonlocal search) ----------------- *
 * Same result as nbx_grid_build(0, home...) + nbx_grid_build(1, halo...) + nbx_search(LOCAL)
 * + nbx_search(NONLOCAL), with the home grid and local list on `stream` and the halo grid
 * and nonlocal list on `side_stream` (two host waits instead of four; the nonlocal work
 * fills the SMs the local work leaves idle).  On return `stream` is ordered after all of it. */
NBX_API int nbx_grid_search_pair(nbx_ctx* ctx, int32_t n_home, const float* x_home_dev, const int32_t* gid_home_dev,
                                 const float lo_home[3], const float size_home[3], int32_t n_halo,
                                 const float* x_halo_dev, const int32_t* gid_halo_dev, const float lo_halo[3],
                                 const float size_halo[3], void* stream, void* side_stream);

/* ---- X buffer op (folded into NBNXM_* in the reference model, pipeline.py:231) ------- *
 * Copy user-order coordinates of grid `grid` into the cluster-ordered xyzq buffer, with
 * the wrap shifts fixed at the last grid build.                                          */
NBX_API int nbx_put_x(nbx_ctx* ctx, int grid, const float* x_dev, void* stream);

/* ---- rolling dynamic prune: KernelKind.PRUNE_ONLY (costs.py:31,162; pipeline.py:233-235)
 * Re-derive the inner list of `list` from its outer list with the current coordinates,
 * processing sci entries e with e % nparts == part (nparts=1: whole list).               */
NBX_API int nbx_prune(nbx_ctx* ctx, int list, int part, int nparts, void* stream);

/* ---- force: KernelKind.NBNXM_LOCAL / NBNXM_NONLOCAL (costs.py:29-30; pipeline.py:231,384)
 * Accumulate forces of the inner list `list` into the cluster force buffers (and, with
 * flags, energies / shift forces into the context's fp64 accumulators).                  */
NBX_API int nbx_force(nbx_ctx* ctx, int list, uint32_t flags, void* stream);

/* ---- F buffer op: KernelKind.REDUCE_FORCES (costs.py:41,172; pipeline.py:250-254,398-401)
 * Write (accumulate != 0: add) grid `grid`'s cluster forces to f_dev[n][3] in the order of
 * the grid-build input, and clear the cluster buffer for the next step.                  */
NBX_API int nbx_get_f(nbx_ctx* ctx, int grid, float* f_dev, int accumulate, void* stream);

/* ---- one non-search MD step as a CUDA graph (pipeline.py:222-235 minus the search step) *
 * nbx_put_x(0) [+ nbx_prune(LOCAL, 0, 1) with NBX_STEP_PRUNE] + nbx_force(LOCAL, F only) +
 * nbx_get_f(0) as one graph launch on `stream`.  Graphs are captured natively per
 * (x_dev, f_dev, what) and refreshed in place after a search / grid build / box or
 * topology change, so the small-box step is not launch-bound.                             */
#define NBX_STEP_PRUNE 1u
NBX_API int nbx_step_graph(nbx_ctx* ctx, const float* x_dev, float* f_dev, uint32_t what, void* stream);

/* ---- NVLink peer-memory DD halo (row e; replaces the halo pulses of pipeline.py:273-278,
 * 363-380 and the reverse force pulses of pipeline.py:403-418 for force-only steps) ----- *
 * One process per GPU on one NVSwitch node.  Each rank allocates an IPC-shared region
 * (flags | published home x | force inbox) for `capacity` home atoms (same on all ranks),
 * exchanges the NBX_PEER_HANDLE_BYTES handles (e.g. an all-gather), opens the others', and
 * after every repartition maps its halo (grid 1 input atom a = owner rank, index in the
 * owner's home order, import shift).  A force-only DD step is then
 *   nbx_peer_put_x (grid-0 X op + publish + signal)  -> local prune/force ->
 *   nbx_peer_halo_x (wait + gather halo x over NVLink into grid 1) -> nonlocal prune ->
 *   nbx_peer_force_nonlocal (j forces red.add'ed into the owners' inboxes + signal) ->
 *   nbx_peer_get_f (wait + grid-0 F op + inbox)
 * with one monotonically increasing `seq` per step, identical on all ranks.  `flags`
 * (NBX_FORCE_ENERGY | NBX_FORCE_VIRIAL, after nbx_clear_energies) make it an energy /
 * virial step: the nonlocal kernel accumulates energies and the halo atoms' x (x) f is
 * summed before the push, the home atoms' before the inbox is added, so nbx_energies
 * (after nbx_peer_get_f here) returns this rank's share and an all-reduce gives the total.
 * Waits are bounded (env NBX_PEER_TIMEOUT_S, default 30): on a timeout the wait kernel
 * records it (nbx_peer_status) and traps -- the context is lost, the step fails loudly.   */
#define NBX_PEER_HANDLE_BYTES 64
NBX_API int nbx_peer_init(nbx_ctx* ctx, int32_t rank, int32_t world, int32_t capacity, void* handle_out);
NBX_API int nbx_peer_open(nbx_ctx* ctx, const void* handles /* world * NBX_PEER_HANDLE_BYTES */);
NBX_API int nbx_peer_set_halo(nbx_ctx* ctx, int32_t n_halo, const int32_t* owner_dev, const int32_t* home_dev,
                              const float* shift_dev /* [n_halo][3] */, void* stream);
NBX_API int nbx_peer_put_x(nbx_ctx* ctx, const float* x_home_dev, uint32_t seq, void* stream);
NBX_API int nbx_peer_halo_x(nbx_ctx* ctx, uint32_t seq, void* stream);
NBX_API int nbx_peer_force_nonlocal(nbx_ctx* ctx, uint32_t seq, uint32_t flags, void* stream);
NBX_API int nbx_peer_get_f(nbx_ctx* ctx, float* f_home_dev, uint32_t seq, uint32_t flags, void* stream);
NBX_API int nbx_peer_status(nbx_ctx* ctx, int32_t* timed_out); /* 0 ok, 1 wait timed out, 2 invalid halo map */

/* ---- device-side DD repartition over the peer regions (the search step of the peer path) --
 * Replaces the host-orchestrated global repartition (every rank reading every atom) with a
 * neighbour-only one: each rank publishes its current home atoms (x, gid), then pulls from the
 * ranks at domain offsets within +-1 (src_rank) the atoms whose wrapped position now lies in its
 * own domain -- its new home set, sorted by global id -- publishes that, and pulls its half-shell
 * halo (off_*: the offsets whose first non-zero component is +1, with the periodic image shift)
 * from the neighbours' new home sets.  Everything is stream-ordered device work with flag
 * waits; the host reads two counts at the end.  Outputs (device, capacity cap_ext):
 * x_ext[0 : n_home] = new home atoms (wrapped), x_ext[n_home : n_home + n_halo] = halo atoms in
 * this rank's frame, gid_ext likewise; owner / home_index / shift [n_halo] = the halo map for
 * nbx_peer_set_halo.  rseq: 1, 2, 3, ... per repartition, identical on all ranks.  Returns
 * NBX_ELIST_OVERFLOW (counts still written) when the new home set exceeds the peer capacity
 * or home + halo exceeds cap_ext: re-create the regions / buffers larger and repartition from
 * global coordinates.  Mirrors the reference's decomposed pair search on home + halo atoms
 * (pipeline.py:329-334).                                                                    */
typedef struct nbx_dd_geom {
    float box[3];          /* periodic box                                                   */
    float dlen[3];         /* domain edge per dimension (box / dims)                         */
    float lo[3], hi[3];    /* this rank's domain                                             */
    float rl;              /* halo width (rlist_outer)                                       */
    int32_t dims[3], coord[3];
    int32_t n_src;         /* ranks this rank's new home atoms can come from (incl. itself)  */
    int32_t src_rank[27];
    int32_t n_off;         /* half-shell import offsets                                      */
    int32_t off_rank[13];
    int32_t off_dir[13][3];
    float off_shift[13][3];
} nbx_dd_geom;
NBX_API int nbx_peer_repartition(nbx_ctx* ctx, const nbx_dd_geom* geom, const float* x_home_dev,
                                 const int32_t* gid_home_dev, int32_t n_home, uint32_t rseq, int32_t cap_ext,
                                 float* x_ext_dev, int32_t* gid_ext_dev, int32_t* owner_dev, int32_t* home_index_dev,
                                 float* shift_dev, int32_t* n_home_out, int32_t* n_halo_out, void* stream);

/* Energies and virial accumulated since the last clear.  Reads grid buffers, so call it
 * after nbx_force and BEFORE nbx_get_f.  e_host[2] = {E_lj, E_coul incl. self term},
 * virial_host[9] = -1/2 sum x (x) f - 1/2 sum s (x) fshift (row-major).  Synchronises.    */
NBX_API int nbx_energies(nbx_ctx* ctx, double* e_host, double* virial_host, void* stream);
NBX_API int nbx_clear_energies(nbx_ctx* ctx, void* stream);

/* ---- introspection (tests, bench) ------------------------------------------------------ */
typedef struct nbx_list_sizes {
    int64_t n_sci;      /* sci entries                                                   */
    int64_t n_cj_outer; /* cj entries of the outer list                                  */
    int64_t n_cj_inner; /* cj entries of the inner list (sum of kept)                    */
    int64_t n_pool;     /* mask-pool entries including the implicit entry 0              */
} nbx_list_sizes;

typedef struct nbx_grid_info {
    int32_t n;      /* atoms                                                              */
    int32_t nslots; /* padded cluster-ordered slots (multiple of 32)                      */
    int32_t ncx, ncy;
} nbx_grid_info;

NBX_API int nbx_grid_info_get(nbx_ctx* ctx, int grid, nbx_grid_info* out);
/* order_host[nslots] (input index or -1), xq_host[nslots*4], type_host[nslots]; any NULL. */
NBX_API int nbx_grid_export(nbx_ctx* ctx, int grid, int32_t* order_host, float* xq_host,
                            int32_t* type_host);
NBX_API int nbx_list_sizes_get(nbx_ctx* ctx, int list, nbx_list_sizes* out);
/* Copy the list to host.  which = 0 outer, 1 inner (inner cj entries are compacted into
 * canonical contiguous order, with sci entries' ranges rewritten accordingly).           */
NBX_API int nbx_list_export(nbx_ctx* ctx, int list, int which, nbx_sci_entry* sci_host,
                            nbx_cj_entry* cj_host, nbx_mask_pool_entry* pool_host);

/* Count, over the inner list, the interacting atom pairs inside the cut-off (interaction
 * bit set, r < rc: the "pair-interactions" of the benchmark metric) and the computed pair
 * slots (32 per active i-cluster x j-cluster tile).  Synchronises `stream`.              */
NBX_API int nbx_count_pairs(nbx_ctx* ctx, int list, int64_t* pairs_out, int64_t* slots_out,
                            void* stream);

/* Measured FP32 FFMA peak of this device (TFLOP/s) from a register-resident FMA loop;
 * used as the roofline denominator.                              */
NBX_API int nbx_fma_peak(nbx_ctx* ctx, double* tflops_out, void* stream);

/* Number of kernel launches this context has issued (bench evidence: gpu_launches).    */
NBX_API int64_t nbx_launch_count(nbx_ctx* ctx);
/* Device allocations the library has made so far (process-wide).  Steady-state steps make none:
 * cudaMalloc / cudaFree contend with NVML (nvidia-smi) polls for the driver lock.          */
NBX_API int64_t nbx_alloc_count(void);

/* ---- domain-decomposition halo (KernelKind.HALO_PACK_UNPACK, costs.py:43,174;
 *      pipeline.py:363-380 coordinates, 403-418 forces) -------------------------------- *
 * pack:   out[k] = x[idx[k]] + shift  (k < n)                                              *
 * unpack_add: f[idx[k]] += in[k]                                                          */
NBX_API int nbx_halo_pack_x(const float* x_dev, const int32_t* idx_dev, int32_t n,
                            const float shift_host[3], float* out_dev, void* stream);
NBX_API int nbx_halo_unpack_add_f(float* f_dev, const int32_t* idx_dev, int32_t n,
                                  const float* in_dev, void* stream);

/* ---- row f4: smooth particle-mesh Ewald and the leap-frog update --------------------- *
 * The reciprocal-space half of the Ewald electrostatics whose real-space half is the
 * EWALD / EWALD_TAB force kernel, as the reference's step submits it after the nonbonded
 * kernels: KernelKind.PME_SPREAD, FFT_3D_FORWARD, PME_SOLVE, FFT_3D_INVERSE, PME_GATHER
 * (costs.py:33-37, pipeline.py:241-246) and GRID_MEMSET (costs.py:42, pipeline.py:256-257).
 * Algorithm and conventions: oracle/pme.py (Essmann et al. 1995, B-spline order 4, the
 * same virial convention as the nonbonded path).  Rectangular boxes; one context per
 * device, stream-ordered, not thread-safe; no CPU fallback.                              */
typedef struct nbx_pme nbx_pme;
typedef struct nbx_pme_params {
    int32_t nk[3];  /* FFT grid (each even, >= 8; oracle/pme.py grid_dims: spacing 0.12 nm) */
    int32_t order;  /* B-spline interpolation order: 4 (GROMACS GPU PME)                   */
    float beta;     /* Ewald splitting coefficient, the real-space kernel's (nbx_consts)   */
    float epsfac;   /* 138.935458 / epsilon_r                                              */
} nbx_pme_params;

NBX_API int nbx_pme_create(int device, const nbx_pme_params* p, nbx_pme** out);
NBX_API int nbx_pme_destroy(nbx_pme* pme);
NBX_API int nbx_pme_set_box(nbx_pme* pme, const float box[3]);
/* Reciprocal-space forces of n charges: f[3a..3a+2] += F_a (device arrays, x and f as
 * [n][3] floats, q as [n]).  flags: NBX_FORCE_ENERGY / NBX_FORCE_VIRIAL accumulate the
 * reciprocal energy / virial into the context (read with nbx_pme_energy).                */
NBX_API int nbx_pme_compute(nbx_pme* pme, int32_t n, const float* x_dev, const float* q_dev, float* f_dev,
                            uint32_t flags, void* stream);
/* The same on the atoms of nonbonded context `ctx`'s grid `grid` (after nbx_put_x or the
 * search step of that step), in its cluster order -- spatially sorted, so the spread and
 * gather touch the charge grid with L2 locality -- with the forces added to the grid's
 * cluster force buffer: the next nbx_get_f returns nonbonded + reciprocal forces.       */
NBX_API int nbx_pme_compute_grid(nbx_pme* pme, nbx_ctx* ctx, int grid, uint32_t flags, void* stream);
/* Reads and clears the accumulated energy and virial (row-major 3x3); syncs `stream`.   */
NBX_API int nbx_pme_energy(nbx_pme* pme, double* e_host, double* virial_host, void* stream);
NBX_API int64_t nbx_pme_launch_count(nbx_pme* pme);
/* One force-only nbx_pme_compute with CUDA events between its stages; ms_host[6] receives
 * the per-stage times (GRID_MEMSET, PME_SPREAD, FFT_3D_FORWARD, PME_SOLVE, FFT_3D_INVERSE,
 * PME_GATHER) for the reference's calibrate samples (costs_adapter.py).  Synchronises.   */
NBX_API int nbx_pme_profile(nbx_pme* pme, int32_t n, const float* x_dev, const float* q_dev, float* f_dev,
                            float* ms_host, void* stream);

/* One non-search step of a GPU-resident Ewald run as one CUDA graph launch: nbx_put_x(0)
 * [+ nbx_prune(LOCAL) with NBX_STEP_PRUNE] + nbx_force(LOCAL) + nbx_pme_compute_grid(0) +
 * nbx_get_f(0) + nbx_leapfrog(x, v, f, inv_mass, dt) (x and v updated in place).  Captured
 * on first use per buffer set / dt and refreshed after searches or box changes.          */
NBX_API int nbx_step_graph_pme(nbx_ctx* ctx, nbx_pme* pme, float* x_dev, float* f_dev, float* v_dev,
                               const float* inv_mass_dev, float dt, uint32_t what, void* stream);

/* Leap-frog update (KernelKind.LEAP_FROG, costs.py:39, pipeline.py:249-251), no
 * constraints: v += f inv_mass dt; x += v dt (device arrays, [n][3] floats).            */
NBX_API int nbx_leapfrog(int32_t n, float* x_dev, float* v_dev, const float* f_dev, const float* inv_mass_dev,
                         float dt, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* NBX_H */
