/* oracle/tsoracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference solve path (tetsolve C++ headers under
 * /root/reference/proj/include/tetsolve). Used only by tests/, by
 * __graft_entry__.smoke() and by bench.py's cpu_baseline leg, as the CHECKER.
 * The product (libtsgpu.so) never links, loads or calls this code.
 *
 * Parity pin: tests/test_oracle_pin.py checks every function below against the
 * unmodified reference compiled in place (oracle/_ref/libtsref.so) — bit-exact
 * for meshes, element matrices, EBE products, assembly, block Jacobi, transfers
 * and aggregation; iteration counts and solutions for inner_pcg / solve /
 * solve_pcge — and against the committed fixtures in tests/golden/.
 */
#ifndef TSORACLE_H
#define TSORACLE_H
#include <stdint.h>
#include "../include/tsgpu.h"

typedef struct {
  int32_t n_nodes, vertex_count, n_elems, n_bc;
  double* coords;      /* [n_nodes][3] */
  int32_t* tets10;     /* [n_elems][10] */
  int32_t* material_id;
  int32_t* bc_node;
  int8_t* bc_axis;
} or_mesh;

typedef struct {
  int32_t n;           /* block rows */
  int32_t* row_ptr;    /* [n+1] */
  int32_t* col_idx;    /* [nnzb] */
  double* blocks;      /* [nnzb][9] (values of T stored as double) */
} or_bcsr;

const char* or_last_error(void);

or_mesh* or_box_mesh(const double* ext, const int32_t* div, int32_t n_if, const double* ifs,
                     int32_t fixed);
or_mesh* or_mesh_from_arrays(int32_t n_nodes, int32_t vertex_count, const double* coords,
                             int32_t n_elems, const int32_t* tets10, const int32_t* mat,
                             int32_t n_bc, const int32_t* bc_node, const int8_t* bc_axis);
void or_mesh_sizes(const or_mesh* m, int32_t* nn, int32_t* nv, int32_t* ne, int32_t* nbc);
void or_mesh_export(const or_mesh* m, double* coords, int32_t* tets10, int32_t* mat,
                    int32_t* bc_node, int8_t* bc_axis);
void or_mesh_mask(const or_mesh* m, uint8_t* mask);
void or_mesh_destroy(or_mesh* m);
int or_material_from_wavespeeds(double vp, double vs, double rho, double* lam, double* mu);

int or_element_matrix(int32_t order, const double* v12, double lam, double mu, double* k);
int or_ebe_apply(const or_mesh* m, int32_t order, int32_t n_mat, const double* lam,
                 const double* mu, const uint8_t* mask, int32_t prec, int32_t workers,
                 const void* u, void* f, int32_t batch);
or_bcsr* or_assemble_bcsr(const or_mesh* m, int32_t order, int32_t n_mat, const double* lam,
                          const double* mu, const uint8_t* mask, int32_t prec);
void or_bcsr_sizes(const or_bcsr* a, int32_t* nrows, int64_t* nnzb);
void or_bcsr_export(const or_bcsr* a, int32_t* row_ptr, int32_t* col_idx, double* blocks);
void or_bcsr_destroy(or_bcsr* a);
int or_bcsr_apply(int32_t nrows, const int32_t* row_ptr, const int32_t* col_idx,
                  const void* blocks, int32_t prec, const void* u, void* f, int32_t batch);
int or_ebe_block_jacobi(const or_mesh* m, int32_t order, int32_t n_mat, const double* lam,
                        const double* mu, const uint8_t* mask, int32_t prec, void* inv);
int or_bj_apply(int32_t n, const void* inv, int32_t prec, const void* r, void* z, int32_t batch);
int or_geo_prolong(const or_mesh* m, int32_t transpose, const float* in, float* out,
                   int32_t batch);
int or_inner_pcg_ebe(const or_mesh* m, int32_t order, int32_t n_mat, const double* lam,
                     const double* mu, const uint8_t* mask, const float* r, float* u,
                     int32_t batch, double tol, int32_t max_iter, int32_t* iters,
                     int32_t* converged);

void* or_levels_create(const or_mesh* m, int32_t n_mat, const double* lam, const double* mu,
                       const ts_solver_config* cfg, int32_t workers, double* setup_s);
void or_levels_sizes(const void* h, int32_t* n0, int32_t* n1, int32_t* n2, int64_t* nnzb2);
void or_levels_export(const void* h, int32_t* agg, int32_t* row_ptr2, int32_t* col_idx2,
                      float* blocks2, uint8_t* mask2, float* m0, float* m1, float* m2);
void or_levels_destroy(void* h);
int or_levels_outer_apply(const void* h, const double* u, double* f, int32_t batch);
int or_solve(const void* h, const double* f, const double* u0, double* u_out, int32_t batch,
             const ts_solver_config* cfg, ts_solve_report* rep);
int or_solve_pcge(const void* h, const double* f, const double* u0, double* u_out,
                  int32_t batch, double tol, int32_t max_iter, ts_solve_report* rep);
void or_rng_sym(uint64_t seed, int64_t n, double* out);
#endif
