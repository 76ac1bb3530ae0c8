/*
 * hf.h — C-ABI of libhf.so, the B200 (sm_100a) implementation of the hot path
 * of the reference package `hyperfree` (arXiv:1904.13131 re-implementation,
 * /root/reference/pkg/src/hyperfree).  Cited as file:line below.
 *
 * The reference is pure Python; its "plugin boundary" is the duck-typed
 * operator API (MatrixFreeTangent.apply/.diagonal, compute_residual,
 * TransferOperator, restrict_solution, the Chebyshev/CG vector algebra).  Each
 * entry point below replaces one of those calls.  INTEGRATION.md shows the
 * ctypes binding a reference maintainer would add.
 *
 * Conventions
 *  - every call returns int status: HF_OK (0) or an HF_ERR_* code; the message
 *    of the last failure on the calling thread is hf_last_error();
 *  - "_dev" pointers are device (CUDA global memory) fp64 arrays; all other
 *    pointers are host memory;
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream);
 *    hot-path calls are asynchronous on that stream, setup calls synchronise;
 *  - vectors use the reference layout: lexicographic lattice nodes (x
 *    fastest), DoF = node * dim + component (fespace.py:3-8);
 *  - the geometry arrays (hf_space_pointers / hf_space_geometry_copy) are SoA:
 *    field f of q-point (cell e, local q) at f * n_qp + e * nq + q; the
 *    tangents' q-point caches are internal (tiled per warp);
 *  - a tangent created with storage_bits = 32 (hf_tangent_create_ex) takes
 *    float x / y arrays in every apply entry point; all others take double;
 *  - handles are not thread-safe; the reduction workspace (hf_ws) must not be
 *    shared by concurrently running streams.
 */
#ifndef HF_H
#define HF_H

#ifdef __cplusplus
extern "C" {
#endif

#define HF_API __attribute__((visibility("default")))
#define HF_ABI_VERSION 1

#define HF_OK 0
#define HF_ERR_ARG 1
#define HF_ERR_CUDA 2
#define HF_ERR_UNSUPPORTED 3
#define HF_ERR_JACOBIAN 4 /* det F <= 0 (material.py:34-40, operators.py:184-188) */
#define HF_ERR_GEOMETRY 5 /* non-positive mapping Jacobian (mesh.py:302-306) */

/* caching strategies, operators.py:72 STRATEGIES */
#define HF_SCALAR 0
#define HF_TENSOR2 1
#define HF_TENSOR4 2

typedef struct hf_space hf_space;       /* one discretisation level (Problem)  */
typedef struct hf_tangent hf_tangent;   /* MatrixFreeTangent                   */
typedef struct hf_transfer hf_transfer; /* TransferOperator                    */
typedef struct hf_ws hf_ws;             /* reduction workspace (one per stream) */
typedef struct hf_coarse hf_coarse;     /* assembled coarsest-level operator    */

typedef struct {
  int code;          /* HF_ERR_JACOBIAN when det F <= 0                        */
  long long element; /* argmin element, as NonPositiveJacobian.element        */
  int qpoint;        /* argmin quadrature point                               */
  double det;        /* min det F                                             */
} hf_error_info;

HF_API const char* hf_last_error(void);
HF_API int hf_abi_version(void);
HF_API int hf_max_degree(int dim);

/* ---- Device block pool (no reference analogue: numpy allocates per call).
 * Every device allocation of the library is pooled: a freed block is kept
 * (after a device synchronisation, the ordering cudaFree gives) and reused
 * for a later request of the same size, so rebuilding the tangent and GMG
 * hierarchy each Newton iteration (solver.py:174) does not go back to the
 * driver.  HF_POOL_MAX_MB caps the pooled bytes (default 32768).
 * hf_pool_release returns every pooled block to the driver; hf_pool_info
 * reports pooled (free) and live (handed-out) bytes. */
HF_API int hf_pool_release(void);
HF_API int hf_pool_info(long long* pooled_bytes, long long* live_bytes);

/* ---- Problem (operators.py:83-116; build_dof_map fespace.py:125-139;
 *      compute_geometry_cache mesh.py:290-307) -------------------------------
 * cells[dim] per-axis cell counts of a structured box lattice (the reference
 * builds cubes, cells[a] = n_cells_per_side); values/derivs_1d are the
 * Basis1D tables (p+1, q) row-major (fespace.py:65-102); vertices
 * (n_vertices, dim) lexicographic (mesh.py:157-167, may be perturbed);
 * mu_el/lam_el per cell (operators.py:101-103); mask per DoF
 * (ConstraintSet.mask, fespace.py:154-167).  Geometry (J^-1, JxW per q-point)
 * is computed on the device. */
HF_API int hf_space_create(int dim, int degree, int nq1, const int* cells, const double* values_1d,
                           const double* derivs_1d, const double* qpoints_1d, const double* qweights_1d,
                           const double* vertices, const double* mu_el, const double* lam_el,
                           const unsigned char* mask, void* stream, hf_space** out);
/* replace the constraint mask (Problem.constraints is mutable) */
HF_API int hf_space_set_mask(hf_space* sp, const unsigned char* mask, void* stream);
HF_API int hf_space_info(const hf_space* sp, long long* n_dofs, long long* n_el, long long* n_qp);
/* device views of GeometryCache.jac_inv (SoA [dim*dim][n_qp]), .jxw, and the mask */
HF_API int hf_space_pointers(const hf_space* sp, const double** jinv_dev, const double** jxw_dev,
                             const unsigned char** mask_dev);
/* copy the geometry into caller-owned device buffers (same SoA layout) */
HF_API int hf_space_geometry_copy(const hf_space* sp, double* jinv_dev, double* jxw_dev, void* stream);
HF_API int hf_space_destroy(hf_space* sp);

/* ---- jacobian_range (operators.py:192-196) ---- */
HF_API int hf_jacobian_range(hf_space* sp, const double* u_dev, void* stream, double* jmin, double* jmax,
                             long long* argmin_element, int* argmin_qpoint);

/* ---- MatrixFreeTangent (operators.py:319-417) -------------------------------
 * create == __init__ + build_cache (292-311); fails with HF_ERR_JACOBIAN and a
 * filled hf_error_info when det F <= 0 (the NonPositiveJacobian path). */
HF_API int hf_tangent_create(hf_space* sp, int strategy, const double* ubar_dev, void* stream, hf_tangent** out,
                             hf_error_info* err);
/* mixed precision: storage_bits = 32 stores the q-point
 * cache in float, and the tangent's x / y vectors are then float arrays too;
 * all arithmetic stays fp64.  storage_bits = 64 is hf_tangent_create.  The
 * diagonal and the element matrices need an fp64 tangent. */
HF_API int hf_tangent_create_ex(hf_space* sp, int strategy, int storage_bits, const double* ubar_dev, void* stream,
                                hf_tangent** out, hf_error_info* err);
/* host-pointer forms for FFI callers holding numpy arrays (the reference-side
 * ctypes binding of INTEGRATION.md): MatrixFreeTangent(problem, u_bar)
 * (operators.py:322-326) from a host u_bar, and .diagonal() (395-410) into a
 * host array; both synchronous */
HF_API int hf_tangent_create_host(hf_space* sp, int strategy, const double* ubar_host, hf_tangent** out,
                                  hf_error_info* err);
HF_API int hf_tangent_diagonal_host(hf_tangent* op, double* d_host);
/* .apply (331-339): y = A x with zero-in / identity-out constrained handling */
HF_API int hf_tangent_apply(hf_tangent* op, const double* x_dev, double* y_dev, void* stream);
/* same, but a no-op while *skip_dev != 0 (device-side early exit for graphs) */
HF_API int hf_tangent_apply_flagged(hf_tangent* op, const double* x_dev, double* y_dev, const int* skip_dev,
                                    void* stream);
/* accumulate only: y += A_loc x over the cells, constrained rows dropped
 * (_local_apply + distribute_local_to_global, 341-393 / fespace.py:307-324) */
HF_API int hf_tangent_apply_raw(hf_tangent* op, const double* x_dev, double* y_dev, const int* skip_dev,
                                void* stream);
/* the cell kernel of .apply only, when the previous kernel on the stream
 * wrote x and y = mask ? x : 0 (hf_cheb_step_fill); programmatic dependent launch */
HF_API int hf_tangent_apply_after_fill(hf_tangent* op, const double* x_dev, double* y_dev, const int* skip_dev,
                                       void* stream);
/* Cell-range form of the accumulate-only apply, for overlapping a multi-GPU
 * interface exchange with interior cells.  Cells are processed
 * in tiles of `cells_per_tile` consecutive cells; tiles [tile0, tile1) are
 * accumulated into y.  mode: 0 plain (y initialised earlier), 1 programmatic
 * dependent of the y = mask ? x : 0 fill, 2 programmatic dependent of a
 * kernel that wrote x and y. */
HF_API int hf_tangent_tiles(const hf_tangent* op, long long* n_tiles, int* cells_per_tile);
HF_API int hf_tangent_apply_tiles(hf_tangent* op, const double* x_dev, double* y_dev, const int* skip_dev,
                                  long long tile0, long long tile1, int mode, void* stream);
/* the same, launched on reserve_sms fewer SMs: the interior tiles of a slab
 * run while the interface exchange (an NCCL kernel on another stream) is in
 * flight, and a persistent block that cannot start beside the NCCL kernel
 * would otherwise finish late by the whole exchange */
HF_API int hf_tangent_apply_tiles_ex(hf_tangent* op, const double* x_dev, double* y_dev, const int* skip_dev,
                                     long long tile0, long long tile1, int mode, int reserve_sms, void* stream);
/* Host-to-host .apply for callers that hold the vectors in host memory (the
 * reference's numpy arrays, operators.py:331-339): y_host = A x_host.  Both
 * buffers must be page-locked (cudaHostAlloc / pinned torch tensors, or
 * registered with hf_host_register).  The cells are cut into `chunks` slabs of
 * last-axis cell layers; the H2D copy of a slab's node planes, its fill + cell
 * kernel, and the D2H copy of finished planes run on three streams, so the
 * copies overlap each other and the kernels.  The pipeline is captured as a
 * CUDA graph on first use per (x_host, y_host, chunks) and replayed after
 * that (a few cached per tangent).  Asynchronous on `stream`: y_host is ready
 * once the stream is synchronised.  Uses device staging vectors owned by the
 * tangent, so calls on one tangent must not run concurrently. */
HF_API int hf_tangent_apply_host(hf_tangent* op, const double* x_host, double* y_host, int chunks, void* stream);
/* The pipeline runs one of four ways: captured as a CUDA graph or enqueued
 * directly, each with the copy directions overlapping or with every D2H held
 * back until the last H2D is done.  On first use per buffer pair all four are
 * timed on this host and the fastest kept (hosts differ: on some, concurrent
 * H2D + D2H is slower than back to back, or a graph with host-memory copy
 * nodes launches slower than direct enqueues).  With HF_E2E_RECAL=1 each
 * buffer pair is timed once more on its 257th call (a first calibration can
 * land in a slow window of the host link).  The calls that calibrate
 * synchronise `stream` (a recalibration first waits for the pair's last step).
 * HF_E2E_ORDER=0..3 forces one variant and turns calibration off.
 * hf_tangent_host_info: the variant kept by the last calibration (0 graph +
 * overlap, 1 graph + serial, 2 direct + overlap, 3 direct + serial, -1 none)
 * and the four measured step times in us (us4[4], 0 if not measured). */
HF_API int hf_tangent_host_info(const hf_tangent* op, int* variant, float* us4);
/* diagnostic: per-warp timestamps of the last apply of an instrumented build
 * (HF_TIMELINE=1 -> libhf_tl.so; HF_ERR_UNSUPPORTED otherwise); n >= 148*16*72 */
HF_API int hf_timeline_fetch(unsigned long long* host, long long n, int clear);
/* Launch-sequence graphs: the host mirror records one V-cycle (multigrid.py:309-351: smoothers,
 * residual, transfers, coarse solve) as a CUDA graph and replays it once per preconditioner
 * application (multigrid.py:350).  hf_graph_begin starts recording the launches made on `stream`
 * (not the default stream; no device allocation may happen until hf_graph_end); hf_graph_end
 * finishes it.  *g == NULL: a new executable graph is created.  *g != NULL (a graph recorded
 * earlier from a launch sequence of the same shape, e.g. the previous Newton iteration's
 * hierarchy): it is updated in place (*updated = 1), or re-created if the shapes differ. */
typedef struct hf_graph hf_graph;
HF_API int hf_graph_begin(void* stream);
HF_API int hf_graph_end(void* stream, hf_graph** g, int* updated);
HF_API int hf_graph_launch(hf_graph* g, void* stream);
HF_API int hf_graph_destroy(hf_graph* g);
/* wait for the work queued on `stream` (e.g. after hf_tangent_apply_host) */
HF_API int hf_stream_synchronize(void* stream);
/* page-lock / release caller-owned host memory (cudaHostRegister) */
HF_API int hf_host_register(void* host_ptr, long long bytes);
HF_API int hf_host_unregister(void* host_ptr);
/* Alternate the direction of successive whole-range applies (forwards,
 * backwards, ...): a sweep then starts on the q-point cache tiles the previous
 * one read last, which a 126 MB L2 may still hold.  Off by default (the
 * single-apply benchmark streams the cache); the multigrid levels turn it on
 * for their smoother sweeps.  Results change only by summation order.
 * Without it a whole-range apply walks the tiles from the last to the first
 * (the vector kernels around it stream forwards, so L2 holds the end of x and
 * y when it starts; environment HF_REVERSE=0 restores forwards).  In either
 * direction the q-point cache is streamed through L2 evict-first and the
 * scatter's reductions are evict-last. */
HF_API int hf_tangent_set_alternate(hf_tangent* op, int on);
/* matrix-based baseline (assemble_matrix / AssembledTangent, operators.py:436-516):
 * vals_dev (n_el, nld, nld) element matrices of a tensor4 tangent, nld = nloc*dim,
 * local DoF n*dim + c; dofs_dev (n_el, nld) their global DoFs (operators.py:474).
 * 3D Q1-Q2 and 2D Q1-Q4. */
HF_API int hf_tangent_assemble_local(hf_tangent* op, double* vals_dev, void* stream);
HF_API int hf_space_cell_dofs(const hf_space* sp, long long* dofs_dev, void* stream);
/* .diagonal (395-410) */
HF_API int hf_tangent_diagonal(hf_tangent* op, double* diag_dev, void* stream);
/* .storage_bytes (412-417), cache.payload_scalars_per_qpoint / payload_nbytes (244-289) */
HF_API int hf_tangent_storage(const hf_tangent* op, long long* storage_bytes, int* payload_scalars,
                              long long* payload_bytes);
HF_API int hf_tangent_destroy(hf_tangent* op);

/* ---- compute_residual (operators.py:205-224) ----
 * traction: host double[dim] or NULL; surf_w_dev: top_surface_weights
 * (operators.py:129-167) per lattice node, required with a traction. */
HF_API int hf_residual(hf_space* sp, const double* u_dev, const double* traction, const double* surf_w_dev,
                       double* out_dev, void* stream, hf_error_info* err);

/* ---- energy (operators.py:227-236): out_dev[0] = sum_q psi(F) JxW, the
 * strain energy without the traction work (the host subtracts
 * traction . (surface_weights u)); HF_ERR_JACOBIAN as hf_residual */
HF_API int hf_energy(hf_space* sp, const double* u_dev, double* out_dev, void* stream, hf_error_info* err);

/* ---- TransferOperator (multigrid.py:27-73) ----
 * interp_1d[a]: host (n_fine_a, n_coarse_a) row-major 1D interpolation matrix
 * of axis a (_interpolation_matrix_1d, multigrid.py:58-73).
 * mode: 0 plain; 1 constrained outputs zeroed (v_cycle r_c[mask]=0,
 * multigrid.py:327); 2 out += result with constrained rows dropped
 * (x += corr after corr[mask]=0, multigrid.py:329-331). */
HF_API int hf_transfer_create(const hf_space* coarse, const hf_space* fine, const double* const* interp_1d,
                              hf_transfer** out);
HF_API int hf_prolong(hf_transfer* t, const double* xc_dev, double* xf_dev, int mode, void* stream);
HF_API int hf_restrict(hf_transfer* t, const double* rf_dev, double* rc_dev, int mode, void* stream);
/* the same with 32/64-bit input and output vectors (fp32 multigrid levels);
 * passes run in fp64 */
HF_API int hf_prolong_ex(hf_transfer* t, const void* xc_dev, int in_bits, void* xf_dev, int out_bits, int mode,
                         void* stream);
HF_API int hf_restrict_ex(hf_transfer* t, const void* rf_dev, int in_bits, void* rc_dev, int out_bits, int mode,
                          void* stream);
HF_API int hf_transfer_destroy(hf_transfer* t);
/* restrict_solution, one level (multigrid.py:76-92); keep_constrained != 0
 * keeps prescribed (non-zero Dirichlet) values */
HF_API int hf_inject(const hf_space* coarse, const hf_space* fine, const double* uf_dev, double* uc_dev,
                     int keep_constrained, void* stream);

/* ---- vector algebra of chebyshev_apply / coarse_solve / cg / Lanczos
 *      (multigrid.py:112-306, solver.py:34-76) ---- */
HF_API int hf_ws_create(hf_ws** out);
HF_API int hf_ws_destroy(hf_ws* w);
/* out_dev[0] = a . b  (deterministic order) */
HF_API int hf_dot(hf_ws* w, long long n, const double* a, const double* b, double* out_dev, const int* skip_dev,
                  void* stream);
/* y = mask ? (x ? x : masked_value) : 0 */
HF_API int hf_fill_masked(long long n, double* y, const double* x, const unsigned char* mask, double masked_value,
                          void* stream);
/* z = inv_d (b - ax); d = first ? z/theta : cd d + cz z; x = (x_zero ? 0 : x) + d
 * (ax == NULL means A x = 0) */
HF_API int hf_cheb_step(long long n, double* x, double* d, const double* b, const double* ax, const double* inv_d,
                        int first, double theta, double cd, double cz, int x_zero, const int* skip_dev, void* stream);
/* hf_cheb_step + the initialisation y_next = mask ? x_new : 0 of the next
 * tangent apply, which is then launched with hf_tangent_apply_after_fill as
 * this kernel's programmatic dependent (y_next may alias ax) */
HF_API int hf_cheb_step_fill(long long n, double* x, double* d, const double* b, const double* ax, const double* inv_d,
                             int first, double theta, double cd, double cz, int x_zero, const int* skip_dev,
                             const unsigned char* mask, double* y_next, void* stream);
/* hf_cheb_step (fill_mask == NULL) or hf_cheb_step_fill on fp64 or fp32
 * vectors (fp_bits), launched as the programmatic dependent of the cell
 * kernel that wrote ax: the tangent apply of the same smoothing step must be
 * the launch immediately before on the stream (multigrid.py:195-204).  The
 * update's blocks load inv_d, b, d and x while that kernel drains and wait for
 * it before they read ax.  x_zero = 0 and ax != NULL by construction. */
HF_API int hf_cheb_step_after_apply(long long n, void* x, void* d, const void* b, const void* ax, const void* inv_d,
                                    int first, double theta, double cd, double cz, const unsigned char* fill_mask,
                                    void* y_next, int fp_bits, void* stream);
/* The Chebyshev step in three-term form (multigrid.py:195-204 with the
 * direction recovered as d = x_k - x_{k-1} instead of stored):
 *   z = inv_d (b - ax); d = first ? z/theta : cd (x_k - x_{k-1}) + cz z;
 *   x_{k+1} = x_k + d, written over x_{k-1} (xo); the caller swaps xk and xo.
 * xk_zero / xprev_zero: that iterate is zero and not read.  One vector write
 * less per step than hf_cheb_step.  fill_mask / y_next as hf_cheb_step_fill;
 * after_apply as hf_cheb_step_after_apply; fp_bits 64 or 32. */
HF_API int hf_cheb3_step(long long n, const void* xk, void* xo, const void* b, const void* ax, const void* inv_d,
                         int first, double theta, double cd, double cz, int xk_zero, int xprev_zero,
                         const unsigned char* fill_mask, void* y_next, int fp_bits, int after_apply, void* stream);
/* r = b - ax; r[mask] = 0 (v_cycle, multigrid.py:324-325) */
HF_API int hf_resid_masked(long long n, double* r, const double* b, const double* ax, const unsigned char* mask,
                           void* stream);
/* scal[out] = ||b - ax||^2; *flag = 1 if sqrt(scal[out]) <= scal[target] (coarse_solve check) */
HF_API int hf_resnorm_check(hf_ws* w, long long n, const double* b, const double* ax, double* scal_dev, int out_idx,
                            int target_idx, int* flag_dev, void* stream);
/* op 0: flag |= sqrt(scal[a]) <= scal[b];  op 1: scal[b] = rel*sqrt(scal[a]), flag = (scal[a] == 0) */
HF_API int hf_scalar_op(int op, double* scal_dev, int a, int b, double rel, int* flag_dev, void* stream);
/* alpha = scal[irz]/scal[ipap]; x += alpha p; r -= alpha ap; scal[irr] = r.r */
HF_API int hf_cg_update_xr(hf_ws* w, long long n, double* x, double* r, const double* p, const double* ap,
                           double* scal_dev, int irz, int ipap, int irr, void* stream);
/* p = z + (scal[irzn]/scal[irz]) p */
HF_API int hf_cg_update_p(long long n, double* p, const double* z, const double* scal_dev, int irzn, int irz,
                          void* stream);
/* hf_cg_update_p + the initialisation y_next = mask ? p_new : 0 of the tangent
 * apply A p that follows (solver.py:58, 73); that apply is then launched with
 * hf_tangent_apply_after_fill as this kernel's programmatic dependent */
HF_API int hf_cg_update_p_fill(long long n, double* p, const double* z, const double* scal, int irzn, int irz,
                               const unsigned char* mask, double* y_next, void* stream);
/* z = inv_d r; out_dev[0] = r . z */
HF_API int hf_jacobi_dot(hf_ws* w, long long n, double* z, const double* r, const double* inv_d, double* out_dev,
                         void* stream);
/* ---- coarse_solve (multigrid.py:255-306) as one persistent kernel ----
 * hf_coarse_create copies the CSR (int32 row pointers / columns, fp64 values)
 * of the coarsest level's assembled tangent, with constrained rows and columns
 * cleared and a unit diagonal (AssembledTangent, operators.py:481-490), i.e.
 * the matrix-free apply's zero-in / identity-out operator.
 * hf_coarse_cheb_solve runs the continuous Chebyshev iteration of
 * _coarse_solve_into in one cooperative launch: x = inv_d b / theta, then up to
 * max_applications - 1 further applications with the residual test
 * ||b - A x|| <= rel_target ||b|| every `degree`-th application; scal_dev[0..2]
 * = ||b||^2, target, last ||b - A x||^2; *flag_dev = 1 if it stopped on the
 * test (or b == 0), 0 if it hit the cap.  d is scratch.  Graph-capturable.
 * A level whose whole matrix and iterate fit one CTA's shared memory runs as
 * a single CTA without grid barriers (HF_COARSE_SINGLE=0 forces the
 * multi-CTA form); the result differs only in the summation order of the
 * residual norm. */
HF_API int hf_coarse_create(long long n, long long nnz, const int* rowptr_dev, const int* col_dev,
                            const double* val_dev, void* stream, hf_coarse** out);
HF_API int hf_coarse_cheb_solve(hf_coarse* c, const double* b, double* x, double* d, const double* inv_d,
                                double theta, double delta, double sigma, double rel_target, int max_applications,
                                int degree, double* scal_dev, int* flag_dev, void* stream);
HF_API int hf_coarse_destroy(hf_coarse* c);
/* The same from a level directly: the sparsity pattern of the space's cell
 * DoF map with the constraint mask applied (constrained rows and columns
 * cleared, unit diagonal; operators.py:471-490) is built once on the host;
 * hf_coarse_update then (asynchronously) refreshes the values from the element
 * matrices of an fp64 tensor4 tangent on that space, each value the sum of its
 * element entries in a fixed order -- no host work per Newton iteration.
 * hf_coarse_clone gives an independent handle (own values and buffers) with
 * the same pattern.  3D Q1-Q2 and 2D Q1-Q4. */
HF_API int hf_coarse_create_space(const hf_space* sp, void* stream, hf_coarse** out);
HF_API int hf_coarse_update(hf_coarse* c, hf_tangent* op, void* stream);
HF_API int hf_coarse_clone(const hf_coarse* src, void* stream, hf_coarse** out);
/* Jacobi-PCG / Lanczos range estimate with device-side scalars
 * (estimate_eigenvalue_range, multigrid.py:112-166): no host round trip per
 * iteration.  scal_dev[4]: [0] rz = r.z (set by hf_jacobi_dot before
 * hf_lanczos_init), [1] pAp, [2] rz_new, [3] beta; state_dev[2]: [0] stop
 * flag, [1] steps recorded; ab_dev[2k] = alpha_k, ab_dev[2k+1] = beta_k.
 * hf_lanczos_init applies the reference's rz > 0 / finite test; each
 * hf_lanczos_step, after ap = A p (skipped while state_dev[0] != 0, e.g.
 * hf_tangent_apply_flagged), does pAp, r -= alpha ap, z = inv_d r, rz_new,
 * the pAp <= 0 / rz_new <= 1e-28 rz / finite tests and p = z + beta p. */
HF_API int hf_lanczos_init(const double* scal_dev, int* state_dev, void* stream);
HF_API int hf_lanczos_step(hf_ws* w, long long n, double* r, double* z, double* p, const double* ap,
                           const double* inv_d, double* scal_dev, double* ab_dev, int* state_dev, void* stream);
/* hf_lanczos_step with the r update, the Jacobi scaling and r.z in one pass
 * and the p update writing y_next = mask ? p : 0, the initialisation of the
 * next iteration's application A p (launched with hf_tangent_apply_after_fill) */
HF_API int hf_lanczos_step_fill(hf_ws* w, long long n, double* r, double* z, double* p, const double* ap,
                                const double* inv_d, double* scal_dev, double* ab_dev, int* state_dev,
                                const unsigned char* mask, double* y_next, void* stream);
/* diagnostic: blocks x threads threads run 8 independent chains of `iters`
 * DFMAs (16 * iters flops per thread) -- the measured fp64 roofline peak */
HF_API int hf_probe_dfma(long long iters, int blocks, int threads, double* sink_dev, void* stream);
/* Box partitions (distributed.py Box; the paper's p4est octants): interface
 * DoFs shared with one neighbour, listed by local index `idx` (the same global
 * order on both ranks).  hf_halo_pack: buf[i] = y[idx[i]]; hf_halo_unpack_add:
 * y[idx[i]] += buf[i] where mask[idx[i]] == 0.  hf_dot_owned: sum of a[i] b[i]
 * over own[i] != 0 (the DoFs this rank owns), deterministic order. */
HF_API int hf_halo_pack(long long n, const int* idx, const double* y, double* buf, void* stream);
HF_API int hf_halo_unpack_add(long long n, const int* idx, double* y, const double* buf, const unsigned char* mask,
                              void* stream);
HF_API int hf_dot_owned(hf_ws* w, long long n, const double* a, const double* b, const unsigned char* own,
                        double* out_dev, void* stream);

/* reverse halo add of a slab interface (multi-GPU; no reference
 * analogue -- the paper's MPI ghost exchange):
 * y[i] += recv[i] where mask[i] == 0 */
HF_API int hf_halo_add(long long n, double* y, const double* recv, const unsigned char* mask, void* stream);
/* fp32-vector versions for mixed-precision levels (arithmetic in fp64;
 * hf_cheb_step_f32 fills y_next = mask ? x : 0 when fill_mask != NULL) */
HF_API int hf_fill_masked_f32(long long n, float* y, const float* x, const unsigned char* mask, double masked_value,
                              void* stream);
HF_API int hf_cheb_step_f32(long long n, float* x, float* d, const float* b, const float* ax, const float* inv_d,
                            int first, double theta, double cd, double cz, int x_zero, const int* skip_dev,
                            const unsigned char* fill_mask, float* y_next, void* stream);
HF_API int hf_resid_masked_f32(long long n, float* r, const float* b, const float* ax, const unsigned char* mask,
                               void* stream);
HF_API int hf_dot_f32(hf_ws* w, long long n, const float* a, const float* b, double* out_dev, void* stream);
HF_API int hf_resnorm_check_f32(hf_ws* w, long long n, const float* b, const float* ax, double* scal, int out_idx,
                                int target_idx, int* flag_dev, void* stream);
/* y = a x + b y */
HF_API int hf_axpby(long long n, double a, const double* x, double b, double* y, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HF_H */
