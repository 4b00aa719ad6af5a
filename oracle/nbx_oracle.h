/*
 * nbx_oracle.h -- CPU oracle of the NBNXM hot path.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load this library, and only as the checker (or the timed CPU baseline).  The product
 * path (libnbx.so) never links or calls it.
 *
 * Parity status: the reference (mdgpusim, /root/reference/pkg) computes no forces, pair
 * lists, energies or virials and pins none in
 * its tests, so this restatement follows the algorithm pinned in DESIGN.md.  It is pinned by
 * (1) analytic two-particle known answers, (2) a float64 all-pairs brute force with exact
 * erfc (oracle/brute.py), (3) Newton-III / virial identities -- not by reference golden
 * vectors, which do not exist ("parity unpinned" against the reference itself).
 *
 * Uses the public nbx.h types so list arrays can be exchanged with the GPU library.
 */
#ifndef NBX_ORACLE_H
#define NBX_ORACLE_H

#include "../include/nbx.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ora_grid ora_grid;
typedef struct ora_list ora_list;

int ora_derive_consts(const nbx_params* p, nbx_consts* out);
/* EWALD_TAB (value, next - value) tables, 2 * c->tab_n floats each (include/nbx.h). */
int ora_ewald_table(const nbx_consts* c, float* ftab, float* vtab);

/* Column grid dimensions: identical formula to the library. */
void ora_grid_dims(const float size[3], double density, int* ncx, int* ncy, float inv_cell[2]);

/* Build a grid from n atoms (x[n][3], gid[n] or NULL = identity) over region lo/size.
 * q/type are GLOBAL arrays indexed by gid.  density = global atoms / box volume.        */
ora_grid* ora_grid_build(int n, const float* x, const int* gid, const float* q_global,
                         const int* type_global, const int* excl_offsets, const int* excl_gids,
                         const float box[3], const int pbc[3], const float lo[3],
                         const float size[3], double density);
void ora_grid_free(ora_grid* g);
int ora_grid_nslots(const ora_grid* g);
int ora_grid_ncx(const ora_grid* g);
int ora_grid_ncy(const ora_grid* g);
double ora_grid_sumq2(const ora_grid* g);
/* order[nslots], xq[nslots*4], type[nslots], gid[nslots]; any may be NULL */
void ora_grid_export(const ora_grid* g, int* order, float* xq, int* type, int* gid);
/* X buffer op: refresh xq from user-order coordinates with the stored wrap shifts. */
void ora_grid_put_x(ora_grid* g, const float* x);

/* Search (mode NBX_LIST_LOCAL: gi == gj half list; NBX_LIST_NONLOCAL: gid rule) at
 * rlist_outer, followed by a full prune to rlist_inner. */
ora_list* ora_search(const ora_grid* gi, const ora_grid* gj, int mode, const nbx_params* p,
                     const float box[3], const int pbc[3]);
void ora_list_free(ora_list* l);
void ora_list_sizes(const ora_list* l, nbx_list_sizes* out);
void ora_list_export(const ora_list* l, int which, nbx_sci_entry* sci, nbx_cj_entry* cj,
                     nbx_mask_pool_entry* pool);
void ora_prune(ora_list* l, const ora_grid* gi, const ora_grid* gj, const nbx_params* p,
               const float box[3], int part, int nparts);

/* Force evaluation over explicit list arrays (so a GPU-built list can be fed in).
 * c6c12 is the plain (c6, c12) table [ntypes*ntypes*2].  f_i/f_j are double [nslots*3]
 * accumulators (may alias when gi == gj); e2 = {E_lj, E_coul} (no self term);
 * fshift = double[27*3].  energy/shift flags as NBX_FORCE_*. nthreads <= 0 = all.       */
/* per-type LJ parameters of the combination rules (pt: 2 * ntypes floats) */
void ora_lj_comb_params(int ljmod, int ntypes, const float* c6c12, float* pt);

void ora_force(int n_sci, const nbx_sci_entry* sci, const nbx_cj_entry* cj,
               const nbx_mask_pool_entry* pool, const float* xq_i, const int* type_i,
               const float* xq_j, const int* type_j, int ntypes, const float* c6c12,
               const nbx_params* p, const float box[3], unsigned flags, double* f_i,
               double* f_j, double* e2, double* fshift, int nthreads);

/* Interacting atom pairs inside the cut-off (interaction bit set, r < rc) of a list. */
long long ora_count_pairs(int n_sci, const nbx_sci_entry* sci, const nbx_cj_entry* cj,
                          const nbx_mask_pool_entry* pool, const float* xq_i, const float* xq_j,
                          const nbx_params* p, const float box[3]);

/* Self energy of the grid's real atoms (Ewald: -epsfac beta/sqrt(pi) sum q^2;
 * RF: -1/2 epsfac c_rf sum q^2). */
double ora_self_energy(const nbx_params* p, double sumq2);

/* F buffer op: f_out[n][3] (+)= f_slots[order^-1]. */
void ora_grid_get_f(const ora_grid* g, const double* f_slots, float* f_out, int accumulate);

/* virial = -1/2 sum_slots x (x) f - 1/2 sum_s svec_s (x) fshift_s  (row-major 3x3) */
void ora_virial(const ora_grid* g, const double* f_slots, const double* fshift,
                const float box[3], double* vir);

/* Ewald rational approximations (fp32 evaluation). */
float ora_ewald_G(float z);
float ora_ewald_H(float z);

#ifdef __cplusplus
}
#endif
#endif
