/* C ABI of the B200-native GaNi cell-problem solver (libfftcell_b200.so).
 *
 * Drop-in boundary for the hot path of the reference package `fftcell`
 * (/root/reference/pkg/src/fftcell).  The reference has no FFI; its boundary is
 * the Python call signature of fftcell.solver / fftcell.homogenize, so every
 * entry point below names the reference function it replaces.  The Python
 * package paper_1311_0089_b200 binds these through ctypes and keeps the
 * reference signatures.
 *
 * Conventions (all entry points):
 *  - plain pointers and sizes; host arrays use the reference layouts exactly:
 *    fields (R, d, *N) row-major, FFT-shifted storage (grid.py:9-20), fp64;
 *    coefficients isotropic (*N) or packed symmetric (d(d+1)/2, *N)
 *    (material.py:30-49);
 *  - host pointers are borrowed for the duration of the call only;
 *  - calls are synchronous; a context is not thread-safe;
 *  - return FC_OK (0) or an FC_E* code; fc_last_error() describes the failure
 *    (thread-local).  Invalid arguments map to the reference's ValueError.
 *  - no CPU fallback: without a usable sm_100 device every call fails with
 *    FC_ECUDA.
 */
#ifndef FFTCELL_B200_H
#define FFTCELL_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FC_OK 0
#define FC_EINVAL 1   /* bad argument (reference: ValueError) */
#define FC_ENOMEM 2   /* device allocation failed */
#define FC_ECUDA 3    /* CUDA runtime error / no device */
#define FC_ENOTSUP 4  /* shape outside the supported envelope */

#define FC_MAX_RHS 8
#define FC_MAX_PHASES 4096 /* distinct tensors of a phase-indexed coefficient field */

/* Coefficient kinds (material.py:147-158 isotropic, material.py:90-145 packed). */
#define FC_COEF_ISOTROPIC 0
#define FC_COEF_PACKED 1

/* Projector selection for fc_project (solver.py:112-122). */
#define FC_PROJ_ORTHOGONAL 0   /* _Projector.apply_orthogonal  */
#define FC_PROJ_GAMMA_REF 1    /* _Projector.apply_gamma_ref   */

/* Solve outcome codes in fc_report.status. */
#define FC_ST_OK 0          /* converged (or stopped with converged flag) */
#define FC_ST_MAXITER 1     /* max_iter exhausted, converged = 0 (solver.py:227-230) */
#define FC_ST_BREAKDOWN 2   /* pAp <= 0 (solver.py:203-212); detail = pAp */
#define FC_ST_DIVERGENT 3   /* fixed-point growth streak (solver.py:275-288) */

typedef struct fc_ctx fc_ctx;

/* Per right-hand-side outcome: mirrors SolveReport (solver.py:77-87). */
typedef struct fc_report {
  int32_t iterations;
  int32_t converged;
  int32_t status;
  int32_t hist_len;   /* entries written to the history row */
  double detail;      /* pAp at breakdown */
} fc_report;

int32_t fc_version(void);
const char* fc_last_error(void);
int32_t fc_device_count(int32_t* count);

/* Plan options (no reference equivalent: kernel selection of this library).
 * Process-wide defaults copied into every context at creation, where the
 * kernels and tile geometry are chosen; existing contexts are unaffected.
 * Defaults are the measured-fastest choices; the alternatives perform the same
 * arithmetic (fin_split: the same sums in another fixed order) and exist for
 * the variant tests and A/B measurements.  Keys:
 *   force_generic (0)  generic shared-memory FFT on every axis
 *   row_threads (0 = auto), mid_threads (0 = auto), outer_threads (0 = auto)  CTA sizes
 *   row_threads_inv (0 = auto)  last sweep CTA size (<= 512): its own row blocks and tensor boxes
 *   row_tma / mid_tma / outer_tma (1)  TMA data movement in the sweeps
 *   outer_seq (-1 = auto)  d = 3 outer sweep one component at a time
 *   inv_pipe (-1 = auto)  persistent double-buffered last sweep
 *   inv_qpre (1)  last sweep: epilogue input staged by a bulk copy issued with the spectrum loads
 *   fin_split (-1 = auto: from 1024 partial sums on)  reductions finalized by a
 *     separate launch (fixed two-level order) instead of the last CTA to arrive;
 *     agrees with the fused finalize to rounding, not bitwise
 *   mid_threads_inv, mid_map, mid_tma_fwd  middle-sweep tiling / thread mapping
 *   aniso_fused (1)  packed coefficients: fused first sweep (0: pointwise kernel + row FFT)
 *   two_field (1)    d = 3, one slab: the outer sweep stores F0^-1 q once, the inverse middle
 *                    sweep rebuilds components 1 and 2 from it (0: three fields; same bits)
 *   fold_fwd (-1)    with two_field: the forward middle sweep stores xi1 v1 + xi2 v2 as one
 *                    field for the outer sweep (-1: for middle pencils >= 243; same bits)
 *   defer_x (1)  CG x update deferred into the next first sweep
 *   fused_exchange (1)  in-process slabs store straight into the peers' buffers
 *   sync_debug (0)  synchronize after every launch
 * Unknown keys return FC_EINVAL. */
int32_t fc_set_plan_option(const char* key, int32_t value);
int32_t fc_reset_plan_options(void);

/* GridSpec + device binding (grid.py:30-83): odd positive shape, Y > 0. */
int32_t fc_create(fc_ctx** out, int32_t dim, const int64_t* shape, const double* half_periods,
                  int32_t device);
void fc_destroy(fc_ctx* ctx);

/* Slab-decomposed context: axis 0 split into nslabs (<= 8) uneven
 * slabs, slab t on devices[t] (devices may repeat: several slabs on one GPU
 * emulate ranks).  Every entry point below accepts it transparently: host
 * arrays keep the full-grid layout, the library scatters / gathers slabs and
 * runs two axis-0 exchanges (peer copies over NVLink) per operator
 * application.  d = 3, any odd axis lengths (register FFT for 3^k and 5 3^k, shared-memory FFT otherwise). */
int32_t fc_create_sharded(fc_ctx** out, int32_t dim, const int64_t* shape, const double* half_periods,
                          int32_t nslabs, const int32_t* devices);

/* One process per GPU: this process owns slab `rank` of `nranks` on `device`;
 * exchanges are NCCL grouped send/recv, reductions an NCCL all-gather of the
 * per-slab sums (summed in rank order on every rank).  unique_id: 128 bytes from
 * fc_nccl_unique_id() on rank 0, broadcast by the caller (torch.distributed).
 * Host arrays keep the full layout; each rank reads / writes its own planes. */
int32_t fc_nccl_unique_id(void* out128);
int32_t fc_create_dist(fc_ctx** out, int32_t dim, const int64_t* shape, const double* half_periods,
                       int32_t nranks, int32_t rank, int32_t device, const void* unique_id);

/* CoefficientField upload (material.py:90-158): count = N (isotropic) or nsym*N (packed). */
int32_t fc_set_coefficients(fc_ctx* ctx, int32_t kind, const double* host, int64_t count);

/* Phase-indexed form of a piecewise-constant packed field (no reference counterpart
 * in storage; the values are those of CoefficientField.components, material.py:90-158):
 * voxel v of the FFT-shifted row-major grid holds the packed tensor
 * table[m * n_phases + labels[v]], m < d(d+1)/2.  count = |N| labels.  The solver
 * reads 2 instead of 8 d(d+1)/2 coefficient bytes per voxel and application; every
 * result is bit-identical to the packed field's.  FC_EINVAL for a label >= n_phases. */
int32_t fc_set_coefficients_indexed(fc_ctx* ctx, int32_t n_phases, const double* table, const uint16_t* labels,
                                    int64_t count);

/* Turn the resident packed field into the indexed form on the device: exact
 * (bitwise) deduplication of the per-voxel tensors, per slab.  *n_phases = the
 * number of distinct tensors (largest slab), 0 when the field is isotropic or has
 * more than max_phases (<= FC_MAX_PHASES) of them and stays as it is.  keep_packed
 * = 0 frees the packed copy (rebuilt on demand by the consumers that need it). */
int32_t fc_compress_coefficients(fc_ctx* ctx, int32_t max_phases, int32_t keep_packed, int32_t* n_phases);

/* Voxel payload straight into HBM (material.py:194-307 format: f64le, row-major,
 * FFT-shifted, component-major): the .bin file streams through pinned staging
 * buffers, never held whole on the host; each slab reads only its planes.  The
 * file must hold exactly (1 or d(d+1)/2) * |N| values (else FC_EINVAL). */
int32_t fc_load_coefficients(fc_ctx* ctx, int32_t kind, const char* bin_path);

/* c_A / C_A of the device coefficient field (CoefficientField.__post_init__,
 * material.py:100-123: closed-form eigenvalue range, material.py:52-87) and the
 * flat index of the first voxel attaining c_A (NULL allowed). */
int32_t fc_coefficient_bounds(fc_ctx* ctx, double* c_A, double* C_A, int64_t* argmin);

/* The solution of the last solve (nrhs fields (d, *N), the layout of
 * save_field, material.py:238-239) streamed from HBM into a .bin payload. */
int32_t fc_save_solution(fc_ctx* ctx, int32_t nrhs, const char* bin_path);

/* apply_A (material.py:182-187): out = A u for nfields fields of shape (d, *N). */
int32_t fc_apply_A(fc_ctx* ctx, const double* u, double* out, int32_t nfields);

/* _Projector(spec, ref).apply_orthogonal / apply_gamma_ref (solver.py:90-122).
 * ref_matrix (d x d, row-major) is required for FC_PROJ_GAMMA_REF. */
int32_t fc_project(fc_ctx* ctx, int32_t which, const double* ref_matrix, const double* u, double* out,
                   int32_t nfields);

/* apply_system (solver.py:125-129): out = G A u with the orthogonal G. */
int32_t fc_apply_system(fc_ctx* ctx, const double* u, double* out, int32_t nfields);

/* solve_cg (solver.py:142-230) for nrhs independent load cases E[nrhs][d].
 *  lam      : scalar reference lambda (> 0) or <= 0 for none (solver.py:162-171)
 *  init     : NULL or warm starts (nrhs, d, *N)
 *  x_out    : NULL (solution stays resident on the device) or (nrhs, d, *N)
 *  rep      : nrhs reports
 *  hist     : NULL or nrhs rows of (max_iter + 1) residual norms
 *  iterates : NULL or room for iterates_cap snapshots of (nrhs, d, *N); returns the
 *             number written in *n_iterates (record_iterates, solver.py:188-189,219-220) */
int32_t fc_solve_cg(fc_ctx* ctx, int32_t nrhs, const double* E, double tol, int32_t max_iter, double lam,
                    const double* init, double* x_out, fc_report* rep, double* hist, double* iterates,
                    int64_t iterates_cap, int64_t* n_iterates);

/* solve_neumann (solver.py:238-295): e <- E - Gamma0 (A - A0) e.
 *  ref_matrix : A0 (d x d)    scale : per-RHS stopping scale max(|E_N|, tiny) (solver.py:258)
 *  x_out      : NULL or the fluctuation e - E, (nrhs, d, *N)
 *  hist       : NULL or nrhs rows of max_iter update norms */
int32_t fc_solve_fixed_point(fc_ctx* ctx, int32_t nrhs, const double* E, double tol, int32_t max_iter,
                             const double* ref_matrix, const double* scale, double* x_out, fc_report* rep,
                             double* hist);

/* Energy matrix of the last solve (homogenize.py:59-67, transforms.py:168-176):
 * out[a][b] = < A (E_a + x_a), E_b + x_b >, a, b < nrhs.  x = NULL uses the
 * solution resident on the device; otherwise x is (nrhs, d, *N) on the host. */
int32_t fc_energy(fc_ctx* ctx, int32_t nrhs, const double* E, const double* x, double* out);

/* Device generator for the BASELINE cfg4 polycrystal: nearest of n_seeds
 * seeds (voxel units on the periodic torus, (n_seeds, 3)) under the minimum image; the
 * coefficient field becomes the grain tensors packed[(n_seeds, 6)].  labels_out (N int32)
 * may be NULL.  Bit-identical to generators.voronoi_labels. */
int32_t fc_generate_voronoi(fc_ctx* ctx, int32_t n_seeds, const double* seeds, const double* packed,
                            int32_t* labels_out);

/* Device generator for the BASELINE cfg5 medium (generators.py:
 * cfg5_sphere_centres / cfg5_two_phase): balls {|o|^2 < radius^2, o integer,
 * |o_a| <= ceil(radius)} around integer centres on the periodic grid.
 * fc_spheres_stamp marks the balls of n centres ((n, 3) int32 voxel indices, in
 * the caller's drawing order) in a device coverage bitmap (allocated and cleared
 * by the first stamp after fc_spheres_finish or context creation) and returns in
 * *covered the number of covered voxels of this context (a slab's planes only;
 * the caller sums over ranks).  fc_spheres_finish turns the bitmap into the
 * isotropic coefficient field (inside: high, outside: low) and frees it.  The
 * result is bit-identical to the host generator for the same centre list. */
int32_t fc_spheres_stamp(fc_ctx* ctx, int32_t n, const int32_t* centres, double radius, int64_t* covered);
int32_t fc_spheres_finish(fc_ctx* ctx, double high, double low);

/* Instrumentation used by bench.py: per-kernel CUDA-event timing and a launch counter. */
int32_t fc_set_profiling(fc_ctx* ctx, int32_t on);
int32_t fc_profile_count(fc_ctx* ctx);
int32_t fc_profile_get(fc_ctx* ctx, int32_t i, char* name, int32_t name_cap, int64_t* launches, double* total_ms);
int32_t fc_profile_reset(fc_ctx* ctx);
int64_t fc_launch_count(fc_ctx* ctx);
/* What the context's plan selected (no reference counterpart; the bench's byte model reads it):
 * "two_field", "fold_fwd", "packed_fused", "n_phases" (0: full field resident), "slabs". */
int32_t fc_plan_info(fc_ctx* ctx, const char* key, int32_t* value);
/* CUDA-event timers on the context's stream: mark slot (0..7); elapsed between two marks (syncs on b). */
int32_t fc_timer_mark(fc_ctx* ctx, int32_t slot);
int32_t fc_timer_elapsed(fc_ctx* ctx, int32_t a, int32_t b, double* ms);

#ifdef __cplusplus
}
#endif

#endif /* FFTCELL_B200_H */
