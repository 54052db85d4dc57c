/*
 * tsgpu.h — C ABI of the B200-native tetsolve solve path (libtsgpu.so).
 *
 * This is the drop-in boundary for the reference's solve path
 * (/root/reference/proj/include/tetsolve, "tetsolve" C++20 headers). Every
 * entry point below replaces one reference interface; the replaced symbol is
 * cited as file:line (relative to /root/reference/proj/include/tetsolve/).
 * The C++ mirror headers in include/tetsolve_b200/ re-expose the reference's
 * own class/function names on top of this ABI, and INTEGRATION.md shows the
 * ctypes / C++ bindings a maintainer would add.
 *
 * Conventions
 *  - Vectors use the reference layout [node][axis][batch]: entry (dof, b) at
 *    data[dof * batch + b], dof = 3 * node + axis (vector_batch.hpp:12-28).
 *  - Construction data (meshes, materials, masks) are HOST pointers.
 *  - *_apply / *_device entry points take DEVICE pointers and a cudaStream_t
 *    passed as void* (NULL = legacy default stream). *_host entry points take
 *    HOST pointers and copy in/out themselves.
 *  - prec is 32 (float) or 64 (double): the reference's T in EbeOperator<T>.
 *  - Every call returns ts_status; on failure ts_last_error() (thread-local)
 *    carries the message. Status codes map 1:1 to the reference's exception
 *    classes (errors.hpp:9-31, solver_config.hpp:111-116).
 *  - There is no CPU fallback: without a usable CUDA device every compute
 *    entry point returns TS_ERR_CUDA.
 */
#ifndef TSGPU_H
#define TSGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  TS_OK = 0,
  TS_ERR_VALIDATION = 1,     /* tetsolve::ValidationError            errors.hpp:18-21 */
  TS_ERR_BREAKDOWN = 2,      /* SolverError: (p,Ap) <= 0             pcg.hpp:105-107, adaptive_cg.hpp:211-212 */
  TS_ERR_NONFINITE = 3,      /* SolverError: NaN residual            pcg.hpp:70,118-120, adaptive_cg.hpp:171 */
  TS_ERR_NO_CONVERGENCE = 4, /* ConvergenceError (carries report)    adaptive_cg.hpp:179-188 */
  TS_ERR_CUDA = 5,
  TS_ERR_NCCL = 6,
  TS_ERR_PARSE = 7           /* ParseError (a ValidationError): "file:line: msg"  errors.hpp:21-25 */
} ts_status;

const char* ts_last_error(void);
const char* ts_version(void);

/* ---------------------------------------------------------------- config */

/* SolverConfig (solver_config.hpp:21-48); defaults via ts_config_default. */
typedef struct {
  double outer_tol;          /* relative residual norm ||r||/||f||   :22 */
  int32_t outer_max_iter;    /* :23 */
  double level_tol[3];       /* level0/1/2 tolerance                 :24-26 */
  int32_t level_max_iter[3]; /* level0/1/2 max update steps          :24-26 */
  int32_t batch_size;        /* CLI/Greens batch width only          :27 */
  int32_t aggregate_target;  /* :28 */
  int32_t residual_history_stride; /* 0 disables history             :29 */
} ts_solver_config;

void ts_config_default(ts_solver_config* cfg);
ts_status ts_config_validate(const ts_solver_config* cfg); /* SolverConfig::validate :31-47 */

/* SolveReport (solver_config.hpp:50-63). Arrays are caller-owned; any may be
 * NULL. history is row-major [history_capacity][batch]. */
typedef struct {
  int32_t converged;
  int32_t outer_iterations;
  int64_t inner_iterations[3];
  double time_setup_s;
  double time_outer_s;
  double time_inner_s[3];
  double time_total_s;
  int32_t batch_size;
  int32_t method;            /* 0 = "amg", 1 = "pcge" */
  int32_t inner_precision;   /* 32 = "float32", 64 = "float64" */
  int32_t history_count;     /* rows written */
  int32_t history_capacity;  /* rows available (in) */
  double* final_rel_residual;/* [batch] */
  int32_t* history_iter;     /* [history_capacity] */
  double* history;           /* [history_capacity][batch] */
} ts_solve_report;

/* ------------------------------------------------------------------ mesh */

/* Host-side mesh container mirroring tetsolve::Mesh (mesh.hpp:26-42):
 * vertices first, tets10 = 4 vertices + 6 edge nodes on edges
 * (0,1),(1,2),(2,0),(0,3),(1,3),(2,3). */
typedef struct ts_mesh ts_mesh;

/* generate_box_mesh (box_mesh.hpp:55-157); fixed_boundary: 0 none,
 * 1 bottom_and_sides, 2 all_clamped (box_mesh.hpp:13-17). Node numbering is
 * identical to the reference (vertices lexicographic z,y,x; edge midpoints in
 * element discovery order). */
ts_status ts_box_mesh(const double extents[3], const int32_t divisions[3],
                      int32_t n_interfaces, const double* layer_interfaces,
                      int32_t fixed_boundary, ts_mesh** out);
ts_status ts_mesh_from_arrays(int32_t n_nodes, int32_t vertex_count, const double* coords,
                              int32_t n_elems, const int32_t* tets10,
                              const int32_t* material_id, int32_t n_dirichlet,
                              const int32_t* bc_node, const int8_t* bc_axis, ts_mesh** out);
ts_status ts_mesh_sizes(const ts_mesh* m, int32_t* n_nodes, int32_t* vertex_count,
                        int32_t* n_elems, int32_t* n_dirichlet);
/* any output pointer may be NULL */
ts_status ts_mesh_export(const ts_mesh* m, double* coords, int32_t* tets10,
                         int32_t* material_id, int32_t* bc_node, int8_t* bc_axis);
/* validate_mesh (mesh.hpp:75-113): TS_ERR_VALIDATION naming the first offending element */
ts_status ts_mesh_validate(const ts_mesh* m);
/* dirichlet_mask (mesh.hpp:150-154): 3*n_nodes bytes */
ts_status ts_mesh_dirichlet_mask(const ts_mesh* m, uint8_t* mask);
void ts_mesh_destroy(ts_mesh* m);

/* ------------------------------------------------------------ file formats */

/* TSMESH 1 text mesh. write: byte-identical to write_mesh (mesh_io.hpp:20-36),
 * through a temporary file renamed over `path` (atomic_write, io_util.hpp:21-49).
 * read: read_mesh (mesh_io.hpp:44-96) — TS_ERR_PARSE "path:line: msg" on a
 * malformed line (same line numbers and messages), then validate_mesh
 * (mesh.hpp:75-113, TS_ERR_VALIDATION naming the first bad element). The read
 * mesh has no Dirichlet entries (they live in the sidecar). */
ts_status ts_mesh_write_tsmesh(const ts_mesh* m, const char* path);
ts_status ts_mesh_read_tsmesh(const char* path, ts_mesh** out);
/* Dirichlet sidecar, "node axis" lines: write_dirichlet / read_dirichlet
 * (mesh_io.hpp:38-42, 98-115); read REPLACES m's Dirichlet list. */
ts_status ts_mesh_write_dirichlet(const ts_mesh* m, const char* path);
ts_status ts_mesh_read_dirichlet(ts_mesh* m, const char* path);
/* TSBMESH 1 binary mesh (this library's format: text header, then raw
 * little-endian coords f64[N][3], tets10 i32[T][10], material i32[T],
 * bc_node i32[D], bc_axis i8[D]); read validates like ts_mesh_read_tsmesh. */
ts_status ts_mesh_write_tsbmesh(const ts_mesh* m, const char* path);
ts_status ts_mesh_read_tsbmesh(const char* path, ts_mesh** out);

/* TSVEC 1 solution file (solution_io.hpp:12-84): u = fp64 [nodes][3][batch].
 * on_device != 0: u is a DEVICE pointer, streamed through pinned staging
 * (PCIe copy of one 64 MB chunk overlapping the file I/O of the next). */
ts_status ts_tsvec_write(const char* path, const double* u, int64_t nodes, int32_t batch, int32_t on_device);
/* header only: dimensions (TS_ERR_PARSE on a bad header, read_solution's checks) */
ts_status ts_tsvec_info(const char* path, int64_t* nodes, int32_t* batch);
/* payload into u (sized by the caller from ts_tsvec_info; mismatch = TS_ERR_VALIDATION) */
ts_status ts_tsvec_read(const char* path, double* u, int64_t nodes, int32_t batch, int32_t on_device);

/* Green's-sweep files. TSFAULT 1 fault faces (write_fault_faces / read_fault_faces,
 * fault.hpp:44-84,414-419); observation lists "x y z axis" (read_observations,
 * greens.hpp:20-44); TSGREENS 1 banks (write_greens_bank / read_greens_bank,
 * greens.hpp:147-222). Readers: call with NULL outputs to get the sizes, then
 * with arrays at least that large; TS_ERR_PARSE as the reference's ParseError. */
ts_status ts_fault_faces_write(const char* path, const int32_t* faces, int32_t n);
ts_status ts_fault_faces_read(const char* path, int32_t* n, int32_t* faces);
ts_status ts_observations_read(const char* path, int32_t* n, double* points, int32_t* axes);
ts_status ts_greens_bank_write(const char* path, int32_t rows, int32_t cols, const double* obs_points,
                               const int32_t* obs_axes, const double* centers, const int32_t* directions,
                               const double* radii, const double* values);
ts_status ts_greens_bank_read(const char* path, int32_t* rows, int32_t* cols, double* obs_points, int32_t* obs_axes,
                              double* centers, int32_t* directions, double* radii, double* values);

/* material_from_wavespeeds (material.hpp:22-34) */
ts_status ts_material_from_wavespeeds(double vp, double vs, double rho, double* lambda,
                                      double* mu);

/* ------------------------------------------------------- EBE operator */

/* EbeOperator<T> (ebe_operator.hpp:29-226), matrix-free
 * f = mask_id(u) + sum_e Q_e K_e Q_e^T (masked u). Immutable after creation;
 * apply may run concurrently on different streams. */
typedef struct ts_ebe ts_ebe;

/* EbeOperator(mesh, order, materials, dof_mask) (ebe_operator.hpp:35-65).
 * materials are given as Lame pairs; dof_mask may be NULL (no constraints)
 * and otherwise has 3 * n_nodes(order) entries. */
ts_status ts_ebe_create(const ts_mesh* mesh, int32_t order, int32_t n_materials,
                        const double* lambda, const double* mu, const uint8_t* dof_mask,
                        int32_t prec, ts_ebe** out);
void ts_ebe_destroy(ts_ebe* op);
ts_status ts_ebe_info(const ts_ebe* op, int32_t* n_nodes, int32_t* n_elements, int32_t* order,
                      int32_t* prec);
/* EbeOperator::apply (ebe_operator.hpp:90-134) on device pointers. */
ts_status ts_ebe_apply(const ts_ebe* op, const void* u, void* f, int32_t batch, void* stream);
/* same, host pointers (H2D + apply + D2H inside). With pinned u and f the
 * transfers overlap the sweep: u rows go up ahead of the first chunk of
 * elements that reads them, finished f rows come back while later chunks
 * sweep (PCIe full duplex); pageable buffers copy, apply, copy. */
ts_status ts_ebe_apply_host(const ts_ebe* op, const void* u, void* f, int32_t batch);
/* chunks of the host-buffer streaming schedule (0 = copy-apply-copy; the
 * schedule is built by the first pinned-host apply) */
ts_status ts_ebe_host_stream_chunks(const ts_ebe* op, int32_t* chunks);
/* extract_block_jacobi(EbeOperator) (ebe_operator.hpp:288-313): inverse 3x3
 * node blocks in the operator precision, written to a HOST array
 * [n_nodes][9] of prec-sized scalars. */
ts_status ts_ebe_block_jacobi_host(const ts_ebe* op, void* inv_blocks);
/* tuning / introspection: number of kernel launches of one apply, and the
 * device time of the last apply's EBE kernel when timing is enabled. */
ts_status ts_ebe_set_timing(ts_ebe* op, int32_t enable);
ts_status ts_ebe_last_kernel_ms(const ts_ebe* op, float* ms);
ts_status ts_ebe_launches_per_apply(const ts_ebe* op, int32_t batch, int32_t* n);
/* the element sweep's unit plan: kind 2 = edge fans, 1 = face pairs, 0 = element-parallel;
 * units, node rows gathered (= scatter-added) per element, fraction of elements in closed
 * fans (pairs: paired fraction), elements per unit */
ts_status ts_ebe_unit_stats(const ts_ebe* op, int32_t* kind, int32_t* units, double* rows_per_element,
                            double* closed_fraction, double* elements_per_unit);
/* deterministic mode (on != 0): the colored sweep (greedy element coloring, build_coloring
 * ebe_operator.hpp:190-214, one launch per color, plain read-add-writes) — every node sums its
 * elements in a fixed order, so results are bitwise reproducible and independent of the batch
 * width (the reference's contract, test_ebe.cpp:254-317). Default off (atomic pair sweep). */
ts_status ts_ebe_set_deterministic(ts_ebe* op, int32_t on);

/* element_matrix (ebe_operator.hpp:78-87): K_e of caller element e in fp64 from the
 * operator's (T-rounded) geometry, row-major [3 npe][3 npe], index 3 local_node + axis
 * (element_stiffness.hpp:13-14). k is a HOST array. */
ts_status ts_ebe_element_matrix(const ts_ebe* op, int32_t e, double* k);
/* assemble_bcsr(EbeOperator<T>) (ebe_operator.hpp:230-284): identity rows at constrained
 * dofs, constrained columns dropped, blocks summed in fp64 in ascending element order and
 * rounded to T. Call with row_ptr = col_idx = blocks = NULL to get *nnzb, then with HOST
 * arrays row_ptr [n_nodes + 1], col_idx [nnzb], blocks [nnzb][9] of the operator precision. */
ts_status ts_ebe_assemble_bcsr(const ts_ebe* op, int64_t* nnzb, int32_t* row_ptr, int32_t* col_idx, void* blocks);

/* ------------------------------------------------ standalone operators (block_csr.hpp,
 * block_jacobi.hpp, prolongation.hpp, pcg.hpp). Created from HOST arrays, held on the
 * device, immutable; *_apply take device pointers and a stream, *_host copy in/out. */

/* BlockCsrMatrix<T> (block_csr.hpp:16-70): n_block_rows, row_ptr [n+1], col_idx [nnzb]
 * (strictly increasing per row, block_csr.hpp:14), blocks [nnzb][9] of prec-sized scalars */
typedef struct ts_bcsr ts_bcsr;
ts_status ts_bcsr_create(int32_t n_block_rows, const int32_t* row_ptr, const int32_t* col_idx, const void* blocks,
                         int32_t prec, ts_bcsr** out);
void ts_bcsr_destroy(ts_bcsr* a);
ts_status ts_bcsr_info(const ts_bcsr* a, int32_t* n_block_rows, int64_t* nnzb, int32_t* prec);
/* BlockCsrMatrix::apply (block_csr.hpp:33-69): fp64 row accumulation in stored order, rounded to T */
ts_status ts_bcsr_apply(const ts_bcsr* a, const void* u, void* f, int32_t batch, void* stream);
ts_status ts_bcsr_apply_host(const ts_bcsr* a, const void* u, void* f, int32_t batch);
/* extract_block_jacobi(BlockCsrMatrix) (block_jacobi.hpp:72-85) -> HOST [n][9] of prec scalars */
ts_status ts_bcsr_block_jacobi_host(const ts_bcsr* a, void* inv_blocks);

/* BlockJacobi<T> (block_jacobi.hpp:15-39): inverse 3x3 node blocks [n][9] */
typedef struct ts_bj ts_bj;
ts_status ts_bj_create(int32_t n_nodes, const void* inv_blocks, int32_t prec, ts_bj** out);
void ts_bj_destroy(ts_bj* m);
/* BlockJacobi::apply (block_jacobi.hpp:22-38): z = M^-1 r, fp64 math rounded to T */
ts_status ts_bj_apply(const ts_bj* m, const void* r, void* z, int32_t batch, void* stream);
ts_status ts_bj_apply_host(const ts_bj* m, const void* r, void* z, int32_t batch);

/* Prolongation (prolongation.hpp:13-62): per fine node CSR row_ptr [n_fine+1], cols / weights;
 * the same weights on every axis. apply: fine = P coarse; restrict: coarse = P^T fine, summed in
 * ascending fine row (the reference's serial scatter order), both in T = prec. */
typedef struct ts_prolong ts_prolong;
ts_status ts_prolong_create(int32_t n_fine, int32_t n_coarse, const int32_t* row_ptr, const int32_t* cols,
                            const double* weights, ts_prolong** out);
void ts_prolong_destroy(ts_prolong* p);
ts_status ts_prolong_apply(const ts_prolong* p, int32_t prec, const void* coarse, void* fine, int32_t batch,
                           void* stream);
ts_status ts_prolong_restrict(const ts_prolong* p, int32_t prec, const void* fine, void* coarse, int32_t batch,
                              void* stream);
/* host buffers: restrict_to_coarse = 0 -> apply (in = coarse), 1 -> restrict (in = fine) */
ts_status ts_prolong_apply_host(const ts_prolong* p, int32_t prec, int32_t restrict_to_coarse, const void* in,
                                void* out, int32_t batch);
/* build_geometric_prolongation (prolongation.hpp:67-98) into HOST arrays row_ptr [N+1],
 * cols / weights [V + 2 (N - V)] */
ts_status ts_geometric_prolongation(const ts_mesh* mesh, int32_t* row_ptr, int32_t* cols, double* weights);

/* inner_pcg (pcg.hpp:52-124) with the block-Jacobi preconditioner m: kind 0 = a ts_ebe,
 * 1 = a ts_bcsr operator (same precision as m). u is the warm start and the result;
 * iterations / converged are InnerStats (pcg.hpp:15-18). Breakdown -> TS_ERR_BREAKDOWN,
 * non-finite residual -> TS_ERR_NONFINITE (SolverError). */
ts_status ts_inner_pcg(int32_t kind, const void* op, const ts_bj* m, const void* r, void* u, int32_t n_nodes,
                       int32_t batch, double tol, int32_t max_iter, int32_t* iterations, int32_t* converged,
                       void* stream);
ts_status ts_inner_pcg_host(int32_t kind, const void* op, const ts_bj* m, const void* r, void* u, int32_t n_nodes,
                            int32_t batch, double tol, int32_t max_iter, int32_t* iterations, int32_t* converged);

/* level-2 setup on HOST arrays (aggregation.hpp:23-170; the same sequential, order-exact code
 * build_solver_levels runs). aggregate_p1: greedy BFS aggregation of the block graph of K1
 * (row_ptr [n+1], col_idx) into agg_of_node [n], *n_aggregates, seeds [n] (first *n_aggregates
 * used; may be NULL). build_level2: A2 = P^T K1 P of fp64 blocks [nnzb][9], constrained fine dofs
 * (fine_mask [3n], NULL = none) dropped, empty coarse diagonals -> 1; call with NULL outputs for
 * *nnzb2, then row_ptr2 [n_aggregates+1], col_idx2 [nnzb2], blocks2 [nnzb2][9]. */
ts_status ts_aggregate_p1(int32_t n, const int32_t* row_ptr, const int32_t* col_idx, int32_t target,
                          int32_t* agg_of_node, int32_t* n_aggregates, int32_t* seeds);
ts_status ts_build_level2(int32_t n, const int32_t* row_ptr, const int32_t* col_idx, const double* blocks,
                          const int32_t* agg_of_node, int32_t n_aggregates, const uint8_t* fine_mask, int64_t* nnzb2,
                          int32_t* row_ptr2, int32_t* col_idx2, double* blocks2);

/* per-column vector operations on HOST VectorBatch data (vector_batch.hpp:43-119), computed
 * on the device: dot_columns (fp64 accumulation) -> out [batch]; axpy y += (T)alpha_b x;
 * xpby p = z + (T)beta_b p; sub out = a - b (n scalars); zero_masked (mask [ndof]); cast_batch */
ts_status ts_dot_columns_host(int32_t prec, int64_t ndof, int32_t batch, const void* x, const void* y, double* out);
ts_status ts_axpy_columns_host(int32_t prec, int64_t ndof, int32_t batch, const double* alpha, const void* x,
                               void* y);
ts_status ts_xpby_columns_host(int32_t prec, int64_t ndof, int32_t batch, const void* z, const double* beta,
                               void* p);
ts_status ts_sub_columns_host(int32_t prec, int64_t n, const void* a, const void* b, void* out);
ts_status ts_zero_masked_host(int32_t prec, int64_t ndof, int32_t batch, void* x, const uint8_t* mask);
ts_status ts_cast_batch_host(int32_t from_prec, int32_t to_prec, int64_t n, const void* x, void* y);

/* ------------------------------------------------------------ level set */

/* SolverLevels / build_solver_levels (adaptive_cg.hpp:27-67), plus
 * build_crust_model (model.hpp:21-29) when dof_mask is NULL (mask derived
 * from the mesh Dirichlet list). */
typedef struct ts_levels ts_levels;
ts_status ts_levels_create(const ts_mesh* mesh, int32_t n_materials, const double* lambda,
                           const double* mu, const uint8_t* dof_mask,
                           const ts_solver_config* cfg, ts_levels** out);
void ts_levels_destroy(ts_levels* lv);
ts_status ts_levels_sizes(const ts_levels* lv, int32_t* n0, int32_t* n1, int32_t* n2,
                          int64_t* nnzb2);
/* setup introspection for parity tests (any pointer may be NULL):
 * agg_of_node [n1], level-2 BCSR row_ptr [n2+1], col_idx [nnzb2],
 * blocks [nnzb2][9] float, mask2 [3*n2], m2 inverse blocks [n2][9] float */
ts_status ts_levels_export(const ts_levels* lv, int32_t* agg_of_node, int32_t* row_ptr2,
                           int32_t* col_idx2, float* blocks2, uint8_t* mask2, float* m2_inv);
/* the fine-level members of SolverLevels (adaptive_cg.hpp:27-36), any pointer may be NULL:
 * m0 [n0][9], m1 [n1][9] float inverse blocks, mask0 [3 n0], mask1 [3 n1], and the
 * aggregation's seed nodes [n2] (Aggregation::seeds, aggregation.hpp:13-17) */
ts_status ts_levels_export_fine(const ts_levels* lv, float* m0_inv, float* m1_inv, uint8_t* mask0, uint8_t* mask1,
                                int32_t* seeds);
/* the operators inside the level set (borrowed, owned by lv) */
ts_status ts_levels_operator(const ts_levels* lv, int32_t which /*0 outer,1 level0,2 level1*/,
                             const ts_ebe** op);

/* the level operator the solve applies (device buffers): 0 outer fp64 tet10, 1 level-0
 * fp32 tet10, 2 level-1 fp32 tet4 — the assembled K1 (float-rounded inputs, fp32 sums)
 * unless TSGPU_L1=ebe; same product as EbeOperator<float> order 1 (ebe_operator.hpp:90) —
 * 3 level-2 Galerkin BCSR (BlockCsrMatrix<float>::apply, block_csr.hpp:33-69) */
ts_status ts_levels_apply(ts_levels* lv, int32_t which, const void* u, void* f, int32_t batch, void* stream);
/* the preconditioner's inter-grid transfers as the solve runs them (fp32 device buffers), each
 * followed by zero_masked on its output level (adaptive_cg.hpp:84-107): 0 u0 = P1 u1, 1 r1 = P1^T r0,
 * 2 u1 = P2 u2, 3 r2 = P2^T r1 (Prolongation::apply / restrict_to_coarse, prolongation.hpp:25-61) */
ts_status ts_levels_transfer(ts_levels* lv, int32_t which, const float* in, float* out, int32_t batch, void* stream);

/* solve (adaptive_cg.hpp:242-263) with host buffers; u_out may alias u0.
 * n_nodes is the node count f, u0 and u_out were sized for: it must equal the
 * level set's (TS_ERR_VALIDATION "solve: dimension mismatch" otherwise, the
 * reference's shape check, ebe_operator.hpp:91-93), so no buffer is over-read
 * or overrun. */
ts_status ts_solve(ts_levels* lv, const double* f, const double* u0, double* u_out,
                   int32_t n_nodes, int32_t batch, const ts_solver_config* cfg, ts_solve_report* rep);
/* solve with device buffers on a stream */
ts_status ts_solve_device(ts_levels* lv, const double* f, const double* u0, double* u_out,
                          int32_t n_nodes, int32_t batch, const ts_solver_config* cfg, ts_solve_report* rep,
                          void* stream);
/* solve_pcge (adaptive_cg.hpp:267-279), host buffers, 64-bit operator; n_nodes as in ts_solve. */
ts_status ts_solve_pcge(const ts_ebe* k, const double* f, const double* u0, double* u_out,
                        int32_t n_nodes, int32_t batch, double tol, int32_t max_iter, ts_solve_report* rep);

/* ------------------------------------------------ partitioned (multi-GPU) solve
 *
 * SURVEY.md §8e. The reference has no distributed path; these
 * entries add the paper's one: the mesh is split into element partitions, one
 * rank per GPU, interface-node partial sums travel between neighbouring
 * partitions inside every EBE product (NCCL send/recv, overlapped with the
 * interior elements) and dot products are all-reduced. Vectors are in each
 * rank's LOCAL node order (ts_dist_local_nodes gives local -> global). */
typedef struct ts_comm ts_comm;
typedef struct ts_thread_world ts_thread_world;
typedef struct ts_dist_levels ts_dist_levels;

/* NCCL communicator, one process per GPU: rank 0 calls ts_comm_nccl_id and
 * broadcasts the 128 bytes (any out-of-band channel, e.g. torch.distributed). */
ts_status ts_comm_nccl_available(char* why, int32_t why_len);
ts_status ts_comm_nccl_id(uint8_t id[128]);
ts_status ts_comm_create_nccl(int32_t nranks, int32_t rank, const uint8_t id[128], int32_t device,
                              ts_comm** out);
/* in-process ranks (one host thread each, any device incl. a shared one) */
ts_status ts_thread_world_create(int32_t nranks, ts_thread_world** out);
void ts_thread_world_destroy(ts_thread_world* w);
ts_status ts_comm_create_thread(ts_thread_world* w, int32_t rank, int32_t device, ts_comm** out);
void ts_comm_destroy(ts_comm* c);
ts_status ts_comm_info(const ts_comm* c, int32_t* rank, int32_t* size, int32_t* device);
/* in-place sum over the ranks of a DEVICE fp64 array (the dot-product all-reduce
 * of the partitioned solve); enqueued on `stream` */
ts_status ts_comm_allreduce_sum(const ts_comm* c, double* data, int64_t n, void* stream);

/* recursive coordinate bisection of element centroids: part[E] in [0, nparts) */
ts_status ts_partition_rcb(const ts_mesh* mesh, int32_t nparts, int32_t* part);

/* host-only plan of one rank (no device needed): sizes, then arrays */
ts_status ts_dist_plan_sizes(const ts_mesh* mesh, const uint8_t* dof_mask, const int32_t* part,
                             int32_t nranks, int32_t rank, int32_t* n_local, int32_t* n_local_vertices,
                             int32_t* n_elems, int32_t* n_nbr, int64_t* n_halo_rows);
/* l2g [n_local], owned [n_local], elems [n_elems], nbr [n_nbr], nbr_rows [n_nbr]
 * (rows per neighbour), halo_rows [n_halo_rows] (local ids, neighbour-major) */
ts_status ts_dist_plan_export(const ts_mesh* mesh, const uint8_t* dof_mask, const int32_t* part,
                              int32_t nranks, int32_t rank, int32_t* l2g, uint8_t* owned, int32_t* elems,
                              int32_t* nbr, int32_t* nbr_rows, int32_t* halo_rows);

/* host-only: level 2 of build_solver_levels (adaptive_cg.hpp:53-65) from the global mesh —
 * K1 assembly, the sequential aggregation, the Galerkin product, its block Jacobi and coarse
 * mask — as the partitioned setup runs it ONCE (on rank 0, then broadcast); sizes out. Used to
 * measure that setup on a host without GPUs (scripts/northstar_setup_host.py). */
ts_status ts_level2_setup_host(const ts_mesh* mesh, int32_t n_materials, const double* lambda, const double* mu,
                               const uint8_t* dof_mask, int32_t aggregate_target, int32_t* n2, int64_t* nnzb2);

/* build_solver_levels (adaptive_cg.hpp:39-67) for this rank's partition of the
 * GLOBAL mesh (every rank passes the same mesh / part); dof_mask NULL =
 * dirichlet_mask(mesh). Level 2 is built once, on rank 0, and broadcast over the comm.
 * The comm must outlive the level set. */
ts_status ts_dist_levels_create(const ts_mesh* mesh, int32_t n_materials, const double* lambda,
                                const double* mu, const uint8_t* dof_mask, const int32_t* part,
                                const ts_solver_config* cfg, ts_comm* comm, ts_dist_levels** out);
void ts_dist_levels_destroy(ts_dist_levels* lv);
ts_status ts_dist_levels_sizes(const ts_dist_levels* lv, int32_t* n_local, int32_t* n_local_vertices,
                               int32_t* n2);
ts_status ts_dist_local_nodes(const ts_dist_levels* lv, int32_t* l2g);
/* this rank's partition: elements, level-0 interface rows (summed over neighbours, i.e. the
 * rows one level-0 product sends), neighbour ranks, and the wall time of ts_dist_levels_create */
ts_status ts_dist_levels_info(const ts_dist_levels* lv, int32_t* n_elements, int64_t* halo_rows0,
                              int32_t* n_neighbours, double* setup_s);
/* solve (adaptive_cg.hpp:242-263) on local vectors; host or device buffers */
ts_status ts_dist_solve(ts_dist_levels* lv, const double* f, const double* u0, double* u_out,
                        int32_t n_local, int32_t batch, const ts_solver_config* cfg, ts_solve_report* rep);
ts_status ts_dist_solve_device(ts_dist_levels* lv, const double* f, const double* u0, double* u_out,
                               int32_t n_local, int32_t batch, const ts_solver_config* cfg, ts_solve_report* rep,
                               void* stream);
/* one partitioned EBE product (device buffers, local order) incl. the halo
 * exchange: which = 0 outer fp64 tet10, 1 level-0 fp32 tet10, 2 level-1 fp32 tet4 */
ts_status ts_dist_ebe_apply(ts_dist_levels* lv, int32_t which, const void* u, void* f, int32_t batch,
                            void* stream);

/* a partitioned EBE operator alone (no level hierarchy), e.g. for the
 * partitioned matvec benchmark: order 1|2, prec 32|64, this rank's partition */
typedef struct ts_dist_ebe ts_dist_ebe;
ts_status ts_dist_ebe_create(const ts_mesh* mesh, int32_t order, int32_t n_materials, const double* lambda,
                             const double* mu, const uint8_t* dof_mask, const int32_t* part, int32_t prec,
                             ts_comm* comm, ts_dist_ebe** out);
void ts_dist_ebe_destroy(ts_dist_ebe* op);
ts_status ts_dist_ebe_info(const ts_dist_ebe* op, int32_t* n_local, int32_t* n_elements, int64_t* halo_rows,
                           int32_t* n_neighbours);
ts_status ts_dist_ebe_local_nodes(const ts_dist_ebe* op, int32_t* l2g);
ts_status ts_dist_ebe_op_apply(ts_dist_ebe* op, const void* u, void* f, int32_t batch, void* stream);
/* the partition's local operator (borrowed; timing controls via ts_ebe_set_timing) */
ts_status ts_dist_ebe_local_operator(ts_dist_ebe* op, ts_ebe** local);

/* ------------------------------------------------ Green's-function sweep
 *
 * find_plane_fault_faces (fault.hpp:86-118) -> build_faulted_model (model.hpp:41-51,
 * split_nodes fault.hpp:140-302) -> compute_greens_bank (greens.hpp:114-145): per batch of
 * cfg->batch_size unit slips (unit_slip_basis fault.hpp:325-343; direction 0 = dip, 1 =
 * strike), slip_to_rhs (fault.hpp:363-388) as ONE multi-case fp64 EBE product on the split
 * mesh, solve() on the base hierarchy, sample_displacement (greens.hpp:50-76). */
typedef struct ts_faulted ts_faulted;
/* faces: NULL to query *n_faces, else [*n_faces][3] base-mesh vertex ids */
ts_status ts_fault_plane_faces(const ts_mesh* mesh, int32_t axis, double coord, const double lo[3],
                               const double hi[3], int32_t* n_faces, int32_t* faces);
ts_status ts_faulted_model_create(const ts_mesh* mesh, int32_t n_materials, const double* lambda,
                                  const double* mu, const int32_t* faces, int32_t n_faces,
                                  const ts_solver_config* cfg, ts_faulted** out);
void ts_faulted_model_destroy(ts_faulted* fm);
ts_status ts_faulted_info(const ts_faulted* fm, int32_t* n_split_nodes, int32_t* split_mesh_nodes,
                          int32_t* n_faces);
/* reconstruct_split_solution (fault.hpp:392-411) for n_slips unit slips: u_base_host
 * [3N][n_slips] (base mesh) -> u_split_host [3 NS][n_slips] (split mesh, NS from
 * ts_faulted_info): every split copy takes its base node's value, plus copies then
 * add half the slip jump and minus copies subtract it */
ts_status ts_reconstruct_split_solution(ts_faulted* fm, int32_t n_slips, const double* centers,
                                        const int32_t* directions, const double* radii, const double* u_base_host,
                                        double* u_split_host);
/* the base model's solver level set (FaultedModel::base.levels), owned by fm */
ts_status ts_faulted_levels(const ts_faulted* fm, ts_levels** levels);
/* right-hand sides of n_slips unit slips: f_host [3N][n_slips] (base mesh) */
ts_status ts_slip_to_rhs(ts_faulted* fm, int32_t n_slips, const double* centers /*[n][3]*/,
                         const int32_t* directions, const double* radii, double* f_host);
/* bank [n_obs][n_slips] row-major; points [n_obs][3], axes 0..2 */
ts_status ts_greens_bank(ts_faulted* fm, int32_t n_slips, const double* centers, const int32_t* directions,
                         const double* radii, int32_t n_obs, const double* points, const int32_t* axes,
                         const ts_solver_config* cfg, double* bank, int32_t* solver_calls,
                         int64_t* outer_iterations);

/* The same bank on a PARTITIONED base mesh (BASELINE configs[4]: the sweep on the
 * configs[3] mesh over the GPUs of one box; greens.hpp:114-145 with the solve of
 * ts_dist_solve). Every rank passes the same global mesh, faces and element
 * partition; each builds its partition's level set, the fault patch and the fault
 * band of the split mesh (slip lifting replicated per rank, no communication),
 * samples the observations whose containing element it owns, and one all-reduce
 * gives every rank the full bank. The comm must outlive the model. */
typedef struct ts_dist_faulted ts_dist_faulted;
ts_status ts_dist_faulted_model_create(const ts_mesh* mesh, int32_t n_materials, const double* lambda,
                                       const double* mu, const int32_t* faces, int32_t n_faces, const int32_t* part,
                                       const ts_solver_config* cfg, ts_comm* comm, ts_dist_faulted** out);
void ts_dist_faulted_model_destroy(ts_dist_faulted* fm);
ts_status ts_dist_faulted_levels(const ts_dist_faulted* fm, ts_dist_levels** levels);
/* this rank's rows [3 n_local][n_slips] of slip_to_rhs (local node order, ts_dist_local_nodes) */
ts_status ts_dist_slip_to_rhs(ts_dist_faulted* fm, int32_t n_slips, const double* centers, const int32_t* directions,
                              const double* radii, double* f_local_host);
/* bank [n_obs][n_slips] row-major, identical on every rank */
ts_status ts_dist_greens_bank(ts_dist_faulted* fm, int32_t n_slips, const double* centers, const int32_t* directions,
                              const double* radii, int32_t n_obs, const double* points, const int32_t* axes,
                              const ts_solver_config* cfg, double* bank, int32_t* solver_calls,
                              int64_t* outer_iterations);

#ifdef __cplusplus
}
#endif

#endif /* TSGPU_H */
