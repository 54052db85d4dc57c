/* oracle/tsoracle.c — TEST INFRASTRUCTURE ONLY: plain-C restatement of the
 * reference solve path, used as the parity CHECKER by tests/, smoke() and
 * bench.py's cpu_baseline leg. Never linked into or called by the product.
 *
 * Every function cites the reference code it restates (paths relative to
 * /root/reference/proj/include/tetsolve/). Floating-point operations are
 * written in the reference's evaluation order and built with
 * -ffp-contract=off, so results are bit-identical to the reference compiled
 * with g++ -O3 on x86-64 (no FMA contraction there either); the pin is checked
 * in tests/test_oracle_pin.py against oracle/_ref/libtsref.so.
 */
#define _POSIX_C_SOURCE 199309L
#include "tsoracle.h"

#include <float.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static __thread char g_err[512];
const char* or_last_error(void) { return g_err; }
static int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}
#define E_VALID 1
#define E_SOLVER 2
#define E_CONV 4

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec + 1e-9 * ts.tv_nsec;
}

/* ------------------------------------------------------------ geometry.hpp */
/* det3 (geometry.hpp:31-35) */
static double det3(const double m[3][3]) {
  return m[0][0] * (m[1][1] * m[2][2] - m[1][2] * m[2][1]) -
         m[0][1] * (m[1][0] * m[2][2] - m[1][2] * m[2][0]) +
         m[0][2] * (m[1][0] * m[2][1] - m[1][1] * m[2][0]);
}
/* invert3 (geometry.hpp:38-52) */
static int invert3(const double m[3][3], double inv[3][3], double min_det) {
  const double d = det3(m);
  if (fabs(d) <= min_det || d == 0.0) return 0;
  const double id = 1.0 / d;
  inv[0][0] = (m[1][1] * m[2][2] - m[1][2] * m[2][1]) * id;
  inv[0][1] = (m[0][2] * m[2][1] - m[0][1] * m[2][2]) * id;
  inv[0][2] = (m[0][1] * m[1][2] - m[0][2] * m[1][1]) * id;
  inv[1][0] = (m[1][2] * m[2][0] - m[1][0] * m[2][2]) * id;
  inv[1][1] = (m[0][0] * m[2][2] - m[0][2] * m[2][0]) * id;
  inv[1][2] = (m[0][2] * m[1][0] - m[0][0] * m[1][2]) * id;
  inv[2][0] = (m[1][0] * m[2][1] - m[1][1] * m[2][0]) * id;
  inv[2][1] = (m[0][1] * m[2][0] - m[0][0] * m[2][1]) * id;
  inv[2][2] = (m[0][0] * m[1][1] - m[0][1] * m[1][0]) * id;
  return 1;
}
/* tet_volume (geometry.hpp:55-58): dot(b-a, cross(c-a, d-a)) / 6 */
static double tet_volume(const double* a, const double* b, const double* c, const double* d) {
  const double u[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]};
  const double v[3] = {c[0] - a[0], c[1] - a[1], c[2] - a[2]};
  const double w[3] = {d[0] - a[0], d[1] - a[1], d[2] - a[2]};
  const double cr[3] = {v[1] * w[2] - v[2] * w[1], v[2] * w[0] - v[0] * w[2],
                        v[0] * w[1] - v[1] * w[0]};
  return (u[0] * cr[0] + u[1] * cr[1] + u[2] * cr[2]) / 6.0;
}

/* ------------------------------------------- std::mt19937_64 (DeterministicRng) */
/* DeterministicRng (verification.hpp:14-19): unit() = (eng() >> 11) * 2^-53 */
typedef struct { uint64_t mt[312]; int i; } mt64;
static void mt64_seed(mt64* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  s->i = 312;
}
static uint64_t mt64_next(mt64* s) {
  if (s->i >= 312) {
    for (int k = 0; k < 312; ++k) {
      const uint64_t y = (s->mt[k] & 0xFFFFFFFF80000000ULL) | (s->mt[(k + 1) % 312] & 0x7FFFFFFFULL);
      s->mt[k] = s->mt[(k + 156) % 312] ^ (y >> 1) ^ ((y & 1ULL) ? 0xB5026F5AA96619E9ULL : 0ULL);
    }
    s->i = 0;
  }
  uint64_t x = s->mt[s->i++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}
void or_rng_sym(uint64_t seed, int64_t n, double* out) {
  mt64 s;
  mt64_seed(&s, seed);
  for (int64_t i = 0; i < n; ++i) out[i] = (double)(mt64_next(&s) >> 11) * 0x1.0p-53 * 2.0 - 1.0;
}

/* ----------------------------------------------------------------- meshes */
static const int kEdgeEnds[6][2] = {{0, 1}, {1, 2}, {2, 0}, {0, 3}, {1, 3}, {2, 3}};

/* open-addressing map (vmin,vmax) -> edge node; plays the role of
 * Mesh::edge_map (mesh.hpp:31) — only discovery order matters for ids */
typedef struct { uint64_t* keys; int32_t* vals; size_t cap, n; } emap;
static void emap_init(emap* m, size_t expect) {
  m->cap = 16;
  while (m->cap < 2 * expect) m->cap <<= 1;
  m->keys = (uint64_t*)malloc(m->cap * sizeof(uint64_t));
  m->vals = (int32_t*)malloc(m->cap * sizeof(int32_t));
  memset(m->keys, 0xff, m->cap * sizeof(uint64_t));
  m->n = 0;
}
static size_t emap_slot(const emap* m, uint64_t k) {
  uint64_t h = k * 0x9E3779B97F4A7C15ULL;
  size_t i = (size_t)(h >> 17) & (m->cap - 1);
  while (m->keys[i] != ~0ULL && m->keys[i] != k) i = (i + 1) & (m->cap - 1);
  return i;
}
static void emap_free(emap* m) { free(m->keys); free(m->vals); }

or_mesh* or_box_mesh(const double* ext, const int32_t* div, int32_t n_if, const double* ifs,
                     int32_t fixed) {
  /* validate_spec (box_mesh.hpp:30-46) */
  for (int a = 0; a < 3; ++a)
    if (ext[a] <= 0.0 || div[a] < 1) { fail(E_VALID, "box mesh spec: bad extents/divisions"); return NULL; }
  double prev = 0.0;
  for (int i = 0; i < n_if; ++i) {
    if (ifs[i] <= prev || ifs[i] >= ext[2]) {
      fail(E_VALID, "box mesh spec: layer interfaces must be strictly increasing and interior to (0, Lz)");
      return NULL;
    }
    prev = ifs[i];
  }
  /* generate_box_mesh (box_mesh.hpp:55-157) */
  const int32_t nx = div[0], ny = div[1], nz = div[2];
  const double hx = ext[0] / nx, hy = ext[1] / ny, hz = ext[2] / nz;
  or_mesh* m = (or_mesh*)calloc(1, sizeof(or_mesh));
  m->vertex_count = (nx + 1) * (ny + 1) * (nz + 1);
  const int64_t ncell = (int64_t)nx * ny * nz;
  m->n_elems = (int32_t)(6 * ncell);
  /* nodes: V + unique edges; upper bound V + 7*V for the Kuhn split */
  size_t cap_nodes = (size_t)m->vertex_count * 8 + 16;
  m->coords = (double*)malloc(cap_nodes * 3 * sizeof(double));
  int32_t nn = 0;
  for (int32_t k = 0; k <= nz; ++k)
    for (int32_t j = 0; j <= ny; ++j)
      for (int32_t i = 0; i <= nx; ++i) {
        m->coords[3 * nn] = i * hx;
        m->coords[3 * nn + 1] = j * hy;
        m->coords[3 * nn + 2] = k * hz;
        ++nn;
      }
  static const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
  m->tets10 = (int32_t*)malloc((size_t)m->n_elems * 10 * sizeof(int32_t));
  m->material_id = (int32_t*)malloc((size_t)m->n_elems * sizeof(int32_t));
  int64_t e = 0;
  for (int32_t k = 0; k < nz; ++k)
    for (int32_t j = 0; j < ny; ++j)
      for (int32_t i = 0; i < nx; ++i)
        for (int p = 0; p < 6; ++p) {
          int32_t corner[4][3] = {{i, j, k}};
          for (int s = 0; s < 3; ++s) {
            for (int a = 0; a < 3; ++a) corner[s + 1][a] = corner[s][a];
            corner[s + 1][perms[p][s]] += 1;
          }
          int32_t v[4];
          for (int s = 0; s < 4; ++s)
            v[s] = corner[s][0] + (nx + 1) * (corner[s][1] + (ny + 1) * corner[s][2]);
          if (tet_volume(m->coords + 3 * v[0], m->coords + 3 * v[1], m->coords + 3 * v[2],
                         m->coords + 3 * v[3]) < 0.0) {
            const int32_t t = v[2];
            v[2] = v[3];
            v[3] = t;
          }
          int32_t* t = m->tets10 + 10 * e;
          for (int s = 0; s < 4; ++s) t[s] = v[s];
          const double zc = (m->coords[3 * v[0] + 2] + m->coords[3 * v[1] + 2] +
                             m->coords[3 * v[2] + 2] + m->coords[3 * v[3] + 2]) / 4.0;
          /* layer_of (box_mesh.hpp:75-82): layer 0 on top */
          int below = 0;
          for (int q = 0; q < n_if; ++q)
            if (zc > ifs[q]) ++below;
          m->material_id[e] = n_if + 1 - 1 - below;
          ++e;
        }
  /* edge midpoints in discovery order (box_mesh.hpp:114-132) */
  emap em;
  emap_init(&em, (size_t)m->vertex_count * 8);
  for (e = 0; e < m->n_elems; ++e) {
    int32_t* t = m->tets10 + 10 * e;
    for (int q = 0; q < 6; ++q) {
      int32_t a = t[kEdgeEnds[q][0]], b = t[kEdgeEnds[q][1]];
      if (a > b) { const int32_t s = a; a = b; b = s; }
      const uint64_t key = ((uint64_t)(uint32_t)a << 32) | (uint32_t)b;
      const size_t s = emap_slot(&em, key);
      int32_t id;
      if (em.keys[s] == ~0ULL) {
        id = nn++;
        const double* ca = m->coords + 3 * (size_t)t[kEdgeEnds[q][0]];
        const double* cb = m->coords + 3 * (size_t)t[kEdgeEnds[q][1]];
        /* 0.5 * (coords[a] + coords[b]) with a, b the UNSORTED element ends */
        for (int c = 0; c < 3; ++c) m->coords[3 * (size_t)id + c] = 0.5 * (ca[c] + cb[c]);
        em.keys[s] = key;
        em.vals[s] = id;
      } else {
        id = em.vals[s];
      }
      t[4 + q] = id;
    }
  }
  emap_free(&em);
  m->n_nodes = nn;
  /* Dirichlet set (box_mesh.hpp:134-155) */
  m->bc_node = (int32_t*)malloc((size_t)nn * 3 * sizeof(int32_t));
  m->bc_axis = (int8_t*)malloc((size_t)nn * 3);
  int32_t nbc = 0;
  if (fixed != 0) {
    double mx = ext[0];
    if (ext[1] > mx) mx = ext[1];
    if (ext[2] > mx) mx = ext[2];
    const double tol = 1e-9 * mx;
    for (int32_t n = 0; n < nn; ++n) {
      const double* c = m->coords + 3 * (size_t)n;
      const int on_bottom = fabs(c[2]) <= tol;
      const int on_top = fabs(c[2] - ext[2]) <= tol;
      const int on_x = fabs(c[0]) <= tol || fabs(c[0] - ext[0]) <= tol;
      const int on_y = fabs(c[1]) <= tol || fabs(c[1] - ext[1]) <= tol;
      if (fixed == 2) {
        if (on_bottom || on_top || on_x || on_y)
          for (int8_t a = 0; a < 3; ++a) { m->bc_node[nbc] = n; m->bc_axis[nbc++] = a; }
        continue;
      }
      if (on_bottom) {
        for (int8_t a = 0; a < 3; ++a) { m->bc_node[nbc] = n; m->bc_axis[nbc++] = a; }
        continue;
      }
      if (on_x) { m->bc_node[nbc] = n; m->bc_axis[nbc++] = 0; }
      if (on_y) { m->bc_node[nbc] = n; m->bc_axis[nbc++] = 1; }
    }
  }
  m->n_bc = nbc;
  return m;
}

or_mesh* or_mesh_from_arrays(int32_t n_nodes, int32_t vertex_count, const double* coords,
                             int32_t n_elems, const int32_t* tets10, const int32_t* mat,
                             int32_t n_bc, const int32_t* bc_node, const int8_t* bc_axis) {
  or_mesh* m = (or_mesh*)calloc(1, sizeof(or_mesh));
  m->n_nodes = n_nodes;
  m->vertex_count = vertex_count;
  m->n_elems = n_elems;
  m->n_bc = n_bc;
  m->coords = (double*)malloc((size_t)n_nodes * 3 * sizeof(double));
  memcpy(m->coords, coords, (size_t)n_nodes * 3 * sizeof(double));
  m->tets10 = (int32_t*)malloc((size_t)n_elems * 10 * sizeof(int32_t));
  memcpy(m->tets10, tets10, (size_t)n_elems * 10 * sizeof(int32_t));
  m->material_id = (int32_t*)malloc((size_t)n_elems * sizeof(int32_t));
  memcpy(m->material_id, mat, (size_t)n_elems * sizeof(int32_t));
  m->bc_node = (int32_t*)malloc((size_t)(n_bc + 1) * sizeof(int32_t));
  m->bc_axis = (int8_t*)malloc((size_t)(n_bc + 1));
  if (n_bc) {
    memcpy(m->bc_node, bc_node, (size_t)n_bc * sizeof(int32_t));
    memcpy(m->bc_axis, bc_axis, (size_t)n_bc);
  }
  return m;
}

void or_mesh_sizes(const or_mesh* m, int32_t* nn, int32_t* nv, int32_t* ne, int32_t* nbc) {
  *nn = m->n_nodes;
  *nv = m->vertex_count;
  *ne = m->n_elems;
  *nbc = m->n_bc;
}
void or_mesh_export(const or_mesh* m, double* coords, int32_t* tets10, int32_t* mat,
                    int32_t* bc_node, int8_t* bc_axis) {
  if (coords) memcpy(coords, m->coords, (size_t)m->n_nodes * 3 * sizeof(double));
  if (tets10) memcpy(tets10, m->tets10, (size_t)m->n_elems * 10 * sizeof(int32_t));
  if (mat) memcpy(mat, m->material_id, (size_t)m->n_elems * sizeof(int32_t));
  if (bc_node) memcpy(bc_node, m->bc_node, (size_t)m->n_bc * sizeof(int32_t));
  if (bc_axis) memcpy(bc_axis, m->bc_axis, (size_t)m->n_bc);
}
/* dirichlet_mask (mesh.hpp:150-154) */
void or_mesh_mask(const or_mesh* m, uint8_t* mask) {
  memset(mask, 0, (size_t)m->n_nodes * 3);
  for (int32_t i = 0; i < m->n_bc; ++i) mask[3 * (size_t)m->bc_node[i] + m->bc_axis[i]] = 1;
}
void or_mesh_destroy(or_mesh* m) {
  if (!m) return;
  free(m->coords); free(m->tets10); free(m->material_id); free(m->bc_node); free(m->bc_axis);
  free(m);
}
/* material_from_wavespeeds (material.hpp:22-34) */
int or_material_from_wavespeeds(double vp, double vs, double rho, double* lam, double* mu) {
  if (vp <= 0.0 || vs <= 0.0 || rho <= 0.0) return fail(E_VALID, "material: vp, vs, rho must be positive");
  if (vp * vp <= 2.0 * vs * vs) return fail(E_VALID, "material: requires vp^2 > 2*vs^2 (lambda must be positive)");
  *mu = rho * vs * vs;
  *lam = rho * (vp * vp - 2.0 * vs * vs);
  return 0;
}

/* ------------------------------------------------------ element_stiffness.hpp */
static const double kQuadA = 0.58541019662496845; /* element_stiffness.hpp:37 */
static const double kQuadB = 0.13819660112501051; /* :38 */
static const double kGradL[4][3] = {{-1, -1, -1}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}}; /* :54 */

/* tet10_ref_gradients (element_stiffness.hpp:64-73) */
static void tet10_ref_gradients(const double xi[3], double g[10][3]) {
  const double l[4] = {1.0 - xi[0] - xi[1] - xi[2], xi[0], xi[1], xi[2]};
  for (int a = 0; a < 4; ++a)
    for (int c = 0; c < 3; ++c) g[a][c] = (4.0 * l[a] - 1.0) * kGradL[a][c];
  for (int e = 0; e < 6; ++e) {
    const int p = kEdgeEnds[e][0], q = kEdgeEnds[e][1];
    for (int c = 0; c < 3; ++c) g[4 + e][c] = 4.0 * (l[p] * kGradL[q][c] + l[q] * kGradL[p][c]);
  }
}
/* tet_geometry (element_stiffness.hpp:77-86) */
static double tet_geometry(const double v[4][3], double inv_jt[3][3]) {
  double j[3][3], inv[3][3];
  for (int c = 0; c < 3; ++c)
    for (int r = 0; r < 3; ++r) j[r][c] = v[c + 1][r] - v[0][r];
  if (!invert3(j, inv, 0.0)) return 0.0;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) inv_jt[r][c] = inv[c][r];
  return det3(j);
}
/* add_block<NN> (element_stiffness.hpp:90-100) */
static void add_block(double* k, int nn, int a, int b, const double ga[3], const double gb[3],
                      double wl, double wm) {
  const double gdot = ga[0] * gb[0] + ga[1] * gb[1] + ga[2] * gb[2];
  double* row0 = k + (3 * a) * (3 * nn) + 3 * b;
  for (int i = 0; i < 3; ++i) {
    double* row = row0 + i * (3 * nn);
    for (int j = 0; j < 3; ++j) row[j] += wl * ga[i] * gb[j] + wm * gb[i] * ga[j];
    row[i] += wm * gdot;
  }
}
/* tet4_stiffness_kernel (element_stiffness.hpp:104-118) */
static double tet4_kernel(const double v[4][3], double lambda, double mu, double* k) {
  double inv_jt[3][3], g[4][3];
  const double detj = tet_geometry(v, inv_jt);
  if (detj == 0.0) return 0.0;
  for (int a = 0; a < 4; ++a)
    for (int r = 0; r < 3; ++r)
      g[a][r] = inv_jt[r][0] * kGradL[a][0] + inv_jt[r][1] * kGradL[a][1] + inv_jt[r][2] * kGradL[a][2];
  memset(k, 0, sizeof(double) * 144);
  const double vol = detj / 6.0;
  for (int a = 0; a < 4; ++a)
    for (int b = 0; b < 4; ++b) add_block(k, 4, a, b, g[a], g[b], vol * lambda, vol * mu);
  return vol;
}
/* tet10_stiffness_kernel (element_stiffness.hpp:123-140), 4-point rule :39-51 */
static double tet10_kernel(const double v[4][3], double lambda, double mu, double* k) {
  double inv_jt[3][3];
  const double detj = tet_geometry(v, inv_jt);
  if (detj == 0.0) return 0.0;
  memset(k, 0, sizeof(double) * 900);
  const double pts[4][3] = {{kQuadB, kQuadB, kQuadB}, {kQuadA, kQuadB, kQuadB},
                            {kQuadB, kQuadA, kQuadB}, {kQuadB, kQuadB, kQuadA}};
  for (int q = 0; q < 4; ++q) {
    double gr[10][3], g[10][3];
    tet10_ref_gradients(pts[q], gr);
    for (int a = 0; a < 10; ++a)
      for (int r = 0; r < 3; ++r)
        g[a][r] = inv_jt[r][0] * gr[a][0] + inv_jt[r][1] * gr[a][1] + inv_jt[r][2] * gr[a][2];
    const double w = (1.0 / 24.0) * detj;
    for (int a = 0; a < 10; ++a)
      for (int b = 0; b < 10; ++b) add_block(k, 10, a, b, g[a], g[b], w * lambda, w * mu);
  }
  return detj / 6.0;
}
int or_element_matrix(int32_t order, const double* v12, double lam, double mu, double* k) {
  double v[4][3];
  for (int a = 0; a < 4; ++a)
    for (int c = 0; c < 3; ++c) v[a][c] = v12[3 * a + c];
  if (order == 1) tet4_kernel(v, lam, mu, k);
  else tet10_kernel(v, lam, mu, k);
  return 0;
}

/* --------------------------------------------------------- ebe_operator.hpp */
typedef struct {
  int order, npe, prec;
  int32_t n_nodes, n_elems;
  int32_t* conn;   /* [E][npe] */
  double* vtx;     /* [E][12], values rounded to T (ebe_operator.hpp:59-62) */
  double* lame;    /* [E][2], rounded to T (:54-55) */
  uint8_t* mask;   /* NULL = unconstrained */
} or_ebe;

static double round_t(double x, int prec) { return prec == 32 ? (double)(float)x : x; }

/* EbeOperator ctor (ebe_operator.hpp:35-65) */
static int ebe_init(or_ebe* op, const or_mesh* m, int order, int32_t n_mat, const double* lam,
                    const double* mu, const uint8_t* mask, int prec) {
  if (order != 1 && order != 2) return fail(E_VALID, "ebe: order must be 1 or 2");
  op->order = order;
  op->npe = order == 1 ? 4 : 10;
  op->prec = prec;
  op->n_nodes = order == 1 ? m->vertex_count : m->n_nodes;
  op->n_elems = m->n_elems;
  op->conn = (int32_t*)malloc((size_t)op->npe * op->n_elems * sizeof(int32_t));
  op->vtx = (double*)malloc((size_t)12 * op->n_elems * sizeof(double));
  op->lame = (double*)malloc((size_t)2 * op->n_elems * sizeof(double));
  op->mask = NULL;
  if (mask) {
    op->mask = (uint8_t*)malloc((size_t)3 * op->n_nodes);
    memcpy(op->mask, mask, (size_t)3 * op->n_nodes);
  }
  for (int32_t e = 0; e < op->n_elems; ++e) {
    const int32_t mid = m->material_id[e];
    if (mid < 0 || mid >= n_mat) return fail(E_VALID, "ebe: element %d references material %d but only %d defined", e, mid, n_mat);
    op->lame[2 * e] = round_t(lam[mid], prec);
    op->lame[2 * e + 1] = round_t(mu[mid], prec);
    for (int a = 0; a < op->npe; ++a) op->conn[(size_t)op->npe * e + a] = m->tets10[10 * (size_t)e + a];
    for (int v = 0; v < 4; ++v)
      for (int c = 0; c < 3; ++c)
        op->vtx[12 * (size_t)e + 3 * v + c] = round_t(m->coords[3 * (size_t)m->tets10[10 * (size_t)e + v] + c], prec);
  }
  return 0;
}
static void ebe_free(or_ebe* op) { free(op->conn); free(op->vtx); free(op->lame); free(op->mask); }

/* element_matrix (ebe_operator.hpp:78-87) */
static void ebe_element_matrix(const or_ebe* op, int32_t e, double* k) {
  double v[4][3];
  for (int a = 0; a < 4; ++a)
    for (int c = 0; c < 3; ++c) v[a][c] = op->vtx[12 * (size_t)e + 3 * a + c];
  if (op->order == 1) tet4_kernel(v, op->lame[2 * e], op->lame[2 * e + 1], k);
  else tet10_kernel(v, op->lame[2 * e], op->lame[2 * e + 1], k);
}

#define LD(p, prec, i) ((prec) == 32 ? (double)((const float*)(p))[i] : ((const double*)(p))[i])

/* apply (ebe_operator.hpp:90-116) serial path + process_element (:143-188) */
static void ebe_apply(const or_ebe* op, const void* u, void* f, int32_t nb) {
  const int64_t nd = 3 * (int64_t)op->n_nodes;
  const int prec = op->prec;
  for (int64_t d = 0; d < nd; ++d)
    for (int32_t b = 0; b < nb; ++b) {
      const int64_t i = d * nb + b;
      if (prec == 32) ((float*)f)[i] = (op->mask && op->mask[d]) ? ((const float*)u)[i] : 0.0f;
      else ((double*)f)[i] = (op->mask && op->mask[d]) ? ((const double*)u)[i] : 0.0;
    }
  const int npe = op->npe, ndl = 3 * npe;
  double* ul = (double*)malloc(sizeof(double) * ndl * nb);
  double* acc = (double*)malloc(sizeof(double) * ndl * nb);
  double k[900];
  for (int32_t e = 0; e < op->n_elems; ++e) {
    const int32_t* conn = op->conn + (size_t)npe * e;
    for (int a = 0; a < npe; ++a)
      for (int i = 0; i < 3; ++i) {
        const int64_t dof = 3 * (int64_t)conn[a] + i;
        double* dst = ul + (size_t)(3 * a + i) * nb;
        if (op->mask && op->mask[dof]) {
          for (int32_t b = 0; b < nb; ++b) dst[b] = 0.0;
        } else {
          for (int32_t b = 0; b < nb; ++b) dst[b] = LD(u, prec, dof * nb + b);
        }
      }
    ebe_element_matrix(op, e, k);
    memset(acc, 0, sizeof(double) * ndl * nb);
    for (int r = 0; r < ndl; ++r) {
      double* arow = acc + (size_t)r * nb;
      const double* krow = k + (size_t)r * ndl;
      for (int c = 0; c < ndl; ++c) {
        const double krc = krow[c];
        const double* uc = ul + (size_t)c * nb;
        for (int32_t b = 0; b < nb; ++b) arow[b] += krc * uc[b];
      }
    }
    for (int a = 0; a < npe; ++a)
      for (int i = 0; i < 3; ++i) {
        const int64_t dof = 3 * (int64_t)conn[a] + i;
        if (op->mask && op->mask[dof]) continue;
        const double* src = acc + (size_t)(3 * a + i) * nb;
        if (prec == 32) {
          float* dst = (float*)f + dof * nb;
          for (int32_t b = 0; b < nb; ++b) dst[b] += (float)src[b];
        } else {
          double* dst = (double*)f + dof * nb;
          for (int32_t b = 0; b < nb; ++b) dst[b] += src[b];
        }
      }
  }
  free(ul);
  free(acc);
}

int or_ebe_apply(const or_mesh* m, int32_t order, int32_t n_mat, const double* lam,
                 const double* mu, const uint8_t* mask, int32_t prec, int32_t workers,
                 const void* u, void* f, int32_t batch) {
  (void)workers; /* the restatement follows the serial path (ebe_operator.hpp:112-115) */
  or_ebe op;
  memset(&op, 0, sizeof op);
  const int rc = ebe_init(&op, m, order, n_mat, lam, mu, mask, prec);
  if (rc == 0) ebe_apply(&op, u, f, batch);
  ebe_free(&op);
  return rc;
}

/* ------------------------------------------------------------ block CSR */
static int cmp_i32(const void* a, const void* b) {
  const int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}
static int32_t entry_of(const or_bcsr* a, int32_t r, int32_t c) {
  int32_t lo = a->row_ptr[r], hi = a->row_ptr[r + 1];
  while (lo < hi) {
    const int32_t mid = (lo + hi) / 2;
    if (a->col_idx[mid] < c) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}
/* assemble_bcsr (ebe_operator.hpp:230-284) */
static or_bcsr* assemble(const or_ebe* op) {
  const int npe = op->npe;
  const int32_t n = op->n_nodes;
  /* adjacency: node -> sorted unique neighbour nodes (:236-251) */
  int32_t* cnt = (int32_t*)calloc((size_t)n + 1, sizeof(int32_t));
  for (int32_t e = 0; e < op->n_elems; ++e)
    for (int a = 0; a < npe; ++a) cnt[op->conn[(size_t)npe * e + a] + 1] += npe;
  for (int32_t i = 0; i < n; ++i) cnt[i + 1] += cnt[i];
  int32_t* buf = (int32_t*)malloc((size_t)cnt[n] * sizeof(int32_t) + 4);
  int32_t* cur = (int32_t*)malloc((size_t)n * sizeof(int32_t) + 4);
  memcpy(cur, cnt, (size_t)n * sizeof(int32_t));
  for (int32_t e = 0; e < op->n_elems; ++e)
    for (int a = 0; a < npe; ++a)
      for (int b = 0; b < npe; ++b) buf[cur[op->conn[(size_t)npe * e + a]]++] = op->conn[(size_t)npe * e + b];
  or_bcsr* m = (or_bcsr*)calloc(1, sizeof(or_bcsr));
  m->n = n;
  m->row_ptr = (int32_t*)calloc((size_t)n + 1, sizeof(int32_t));
  int32_t w = 0;
  for (int32_t r = 0; r < n; ++r) {
    int32_t* row = buf + cnt[r];
    const int32_t len = cnt[r + 1] - cnt[r];
    qsort(row, (size_t)len, sizeof(int32_t), cmp_i32);
    int32_t u = 0;
    for (int32_t i = 0; i < len; ++i)
      if (u == 0 || row[i] != row[u - 1]) row[u++] = row[i];
    for (int32_t i = 0; i < u; ++i) buf[w + i] = row[i];
    w += u;
    m->row_ptr[r + 1] = w;
  }
  m->col_idx = (int32_t*)malloc((size_t)w * sizeof(int32_t) + 4);
  memcpy(m->col_idx, buf, (size_t)w * sizeof(int32_t));
  free(buf);
  free(cur);
  free(cnt);
  m->blocks = (double*)calloc((size_t)w * 9 + 1, sizeof(double));
  double k[900];
  const uint8_t* mask = op->mask;
  for (int32_t e = 0; e < op->n_elems; ++e) {
    ebe_element_matrix(op, e, k);
    for (int a = 0; a < npe; ++a)
      for (int b = 0; b < npe; ++b) {
        const int32_t ga = op->conn[(size_t)npe * e + a], gb = op->conn[(size_t)npe * e + b];
        double* blk = m->blocks + 9 * (size_t)entry_of(m, ga, gb);
        for (int i = 0; i < 3; ++i) {
          if (mask && mask[3 * (size_t)ga + i]) continue;
          for (int j = 0; j < 3; ++j) {
            if (mask && mask[3 * (size_t)gb + j]) continue;
            blk[3 * i + j] += k[(3 * a + i) * 3 * npe + 3 * b + j];
          }
        }
      }
  }
  if (mask)
    for (int32_t r = 0; r < n; ++r)
      for (int i = 0; i < 3; ++i)
        if (mask[3 * (size_t)r + i]) m->blocks[9 * (size_t)entry_of(m, r, r) + 4 * i] = 1.0;
  for (size_t q = 0; q < (size_t)w * 9; ++q) m->blocks[q] = round_t(m->blocks[q], op->prec);
  return m;
}
or_bcsr* or_assemble_bcsr(const or_mesh* mesh, int32_t order, int32_t n_mat, const double* lam,
                          const double* mu, const uint8_t* mask, int32_t prec) {
  or_ebe op;
  memset(&op, 0, sizeof op);
  if (ebe_init(&op, mesh, order, n_mat, lam, mu, mask, prec)) { ebe_free(&op); return NULL; }
  or_bcsr* a = assemble(&op);
  ebe_free(&op);
  return a;
}
void or_bcsr_sizes(const or_bcsr* a, int32_t* nrows, int64_t* nnzb) {
  *nrows = a->n;
  *nnzb = a->row_ptr[a->n];
}
void or_bcsr_export(const or_bcsr* a, int32_t* row_ptr, int32_t* col_idx, double* blocks) {
  memcpy(row_ptr, a->row_ptr, ((size_t)a->n + 1) * sizeof(int32_t));
  memcpy(col_idx, a->col_idx, (size_t)a->row_ptr[a->n] * sizeof(int32_t));
  memcpy(blocks, a->blocks, (size_t)a->row_ptr[a->n] * 9 * sizeof(double));
}
static void bcsr_free(or_bcsr* a) {
  if (!a) return;
  free(a->row_ptr); free(a->col_idx); free(a->blocks);
}
void or_bcsr_destroy(or_bcsr* a) { bcsr_free(a); free(a); }

/* BlockCsrMatrix<T>::apply (block_csr.hpp:33-69); blocks hold T values */
static void bcsr_apply_t(int32_t nrows, const int32_t* row_ptr, const int32_t* col_idx,
                         const double* blocks, int prec, const void* u, void* f, int32_t nb) {
  double* acc = (double*)malloc(sizeof(double) * 3 * nb);
  for (int32_t r = 0; r < nrows; ++r) {
    for (int32_t i = 0; i < 3 * nb; ++i) acc[i] = 0.0;
    for (int32_t e = row_ptr[r]; e < row_ptr[r + 1]; ++e) {
      const double* blk = blocks + 9 * (size_t)e;
      const int64_t uc = 3 * (int64_t)col_idx[e] * nb;
      for (int i = 0; i < 3; ++i) {
        const double b0 = blk[3 * i], b1 = blk[3 * i + 1], b2 = blk[3 * i + 2];
        double* a = acc + (size_t)i * nb;
        for (int32_t b = 0; b < nb; ++b)
          a[b] += b0 * LD(u, prec, uc + b) + b1 * LD(u, prec, uc + b + nb) + b2 * LD(u, prec, uc + b + 2 * nb);
      }
    }
    const int64_t fr = 3 * (int64_t)r * nb;
    for (int64_t i = 0; i < 3 * (int64_t)nb; ++i) {
      if (prec == 32) ((float*)f)[fr + i] = (float)acc[i];
      else ((double*)f)[fr + i] = acc[i];
    }
  }
  free(acc);
}
int or_bcsr_apply(int32_t nrows, const int32_t* row_ptr, const int32_t* col_idx,
                  const void* blocks, int32_t prec, const void* u, void* f, int32_t batch) {
  const int64_t nnzb = row_ptr[nrows];
  double* bl = (double*)malloc(sizeof(double) * 9 * (size_t)nnzb + 8);
  for (int64_t q = 0; q < 9 * nnzb; ++q) bl[q] = LD(blocks, prec, q);
  bcsr_apply_t(nrows, row_ptr, col_idx, bl, prec, u, f, batch);
  free(bl);
  return 0;
}

/* --------------------------------------------------------- block_jacobi.hpp */
/* invert_node_block (block_jacobi.hpp:45-66); result rounded to T */
static int invert_node_block(double blk[3][3], const uint8_t* dof_mask, int32_t node, int prec,
                             double* out) {
  if (dof_mask)
    for (int i = 0; i < 3; ++i)
      if (dof_mask[i]) {
        for (int j = 0; j < 3; ++j) blk[i][j] = blk[j][i] = 0.0;
        blk[i][i] = 1.0;
      }
  double inv[3][3], scale = 0.0;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      if (fabs(blk[i][j]) > scale) scale = fabs(blk[i][j]);
  if (scale == 0.0 || !invert3(blk, inv, 1e-300))
    return fail(E_VALID, "block jacobi: singular diagonal block at node %d", node);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) out[3 * i + j] = round_t(inv[i][j], prec);
  return 0;
}
/* extract_block_jacobi(EbeOperator) (ebe_operator.hpp:288-313); inv as double(T) */
static int ebe_bj(const or_ebe* op, double* inv) {
  const int npe = op->npe;
  double* diag = (double*)calloc((size_t)op->n_nodes * 9, sizeof(double));
  double k[900];
  for (int32_t e = 0; e < op->n_elems; ++e) {
    ebe_element_matrix(op, e, k);
    for (int a = 0; a < npe; ++a) {
      const int32_t g = op->conn[(size_t)npe * e + a];
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) diag[9 * (size_t)g + 3 * i + j] += k[(3 * a + i) * 3 * npe + 3 * a + j];
    }
  }
  int rc = 0;
  for (int32_t node = 0; node < op->n_nodes && rc == 0; ++node) {
    double blk[3][3];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) blk[i][j] = diag[9 * (size_t)node + 3 * i + j];
    rc = invert_node_block(blk, op->mask ? op->mask + 3 * (size_t)node : NULL, node, op->prec,
                           inv + 9 * (size_t)node);
  }
  free(diag);
  return rc;
}
/* extract_block_jacobi(BlockCsrMatrix) (block_jacobi.hpp:72-85) */
static int bcsr_bj(const or_bcsr* a, int prec, double* inv) {
  for (int32_t r = 0; r < a->n; ++r) {
    double d[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    for (int32_t e = a->row_ptr[r]; e < a->row_ptr[r + 1]; ++e)
      if (a->col_idx[e] == r) {
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) d[i][j] = a->blocks[9 * (size_t)e + 3 * i + j];
        break;
      }
    const int rc = invert_node_block(d, NULL, r, prec, inv + 9 * (size_t)r);
    if (rc) return rc;
  }
  return 0;
}
int or_ebe_block_jacobi(const or_mesh* m, int32_t order, int32_t n_mat, const double* lam,
                        const double* mu, const uint8_t* mask, int32_t prec, void* inv) {
  or_ebe op;
  memset(&op, 0, sizeof op);
  int rc = ebe_init(&op, m, order, n_mat, lam, mu, mask, prec);
  if (rc == 0) {
    double* d = (double*)malloc(sizeof(double) * 9 * (size_t)op.n_nodes);
    rc = ebe_bj(&op, d);
    for (size_t q = 0; q < 9 * (size_t)op.n_nodes; ++q) {
      if (prec == 32) ((float*)inv)[q] = (float)d[q];
      else ((double*)inv)[q] = d[q];
    }
    free(d);
  }
  ebe_free(&op);
  return rc;
}
/* BlockJacobi<T>::apply (block_jacobi.hpp:22-38): fp64 math, rounded to T */
static void bj_apply_t(int32_t n, const double* m, int prec, const void* r, void* z, int32_t nb) {
  for (int32_t node = 0; node < n; ++node) {
    const double* mm = m + 9 * (size_t)node;
    const int64_t base = 3 * (int64_t)node * nb;
    for (int i = 0; i < 3; ++i)
      for (int32_t b = 0; b < nb; ++b) {
        const double v = mm[3 * i] * LD(r, prec, base + b) + mm[3 * i + 1] * LD(r, prec, base + nb + b) +
                         mm[3 * i + 2] * LD(r, prec, base + 2 * nb + b);
        if (prec == 32) ((float*)z)[base + i * nb + b] = (float)v;
        else ((double*)z)[base + i * nb + b] = v;
      }
  }
}
int or_bj_apply(int32_t n, const void* inv, int32_t prec, const void* r, void* z, int32_t batch) {
  double* m = (double*)malloc(sizeof(double) * 9 * (size_t)n);
  for (size_t q = 0; q < 9 * (size_t)n; ++q) m[q] = LD(inv, prec, q);
  bj_apply_t(n, m, prec, r, z, batch);
  free(m);
  return 0;
}

/* --------------------------------------------------------- prolongation.hpp */
typedef struct {
  int32_t n_fine, n_coarse;
  int32_t* row_ptr;
  int32_t* cols;
  double* weights;
} or_prolong;
/* Prolongation::apply<float> (prolongation.hpp:25-40) */
static void prolong_apply(const or_prolong* p, const float* coarse, float* fine, int32_t nb) {
  for (int32_t fn = 0; fn < p->n_fine; ++fn) {
    float* out = fine + 3 * (int64_t)fn * nb;
    for (int64_t i = 0; i < 3 * (int64_t)nb; ++i) out[i] = 0.0f;
    for (int32_t e = p->row_ptr[fn]; e < p->row_ptr[fn + 1]; ++e) {
      const float w = (float)p->weights[e];
      const float* in = coarse + 3 * (int64_t)p->cols[e] * nb;
      for (int i = 0; i < 3; ++i)
        for (int32_t b = 0; b < nb; ++b) out[i * nb + b] += w * in[i * nb + b];
    }
  }
}
/* Prolongation::restrict_to_coarse<float> (prolongation.hpp:44-61) */
static void prolong_restrict(const or_prolong* p, const float* fine, float* coarse, int32_t nb) {
  memset(coarse, 0, sizeof(float) * 3 * (size_t)p->n_coarse * nb);
  for (int32_t fn = 0; fn < p->n_fine; ++fn) {
    const float* in = fine + 3 * (int64_t)fn * nb;
    for (int32_t e = p->row_ptr[fn]; e < p->row_ptr[fn + 1]; ++e) {
      const float w = (float)p->weights[e];
      float* out = coarse + 3 * (int64_t)p->cols[e] * nb;
      for (int i = 0; i < 3; ++i)
        for (int32_t b = 0; b < nb; ++b) out[i * nb + b] += w * in[i * nb + b];
    }
  }
}
static void prolong_free(or_prolong* p) { free(p->row_ptr); free(p->cols); free(p->weights); }
/* build_geometric_prolongation (prolongation.hpp:67-98); edge endpoints
 * (vmin, vmax) as stored in Mesh::edge_map */
static int build_geo(const or_mesh* m, or_prolong* p) {
  p->n_fine = m->n_nodes;
  p->n_coarse = m->vertex_count;
  int32_t* ends = (int32_t*)malloc(sizeof(int32_t) * 2 * (size_t)m->n_nodes);
  for (size_t i = 0; i < 2 * (size_t)m->n_nodes; ++i) ends[i] = -1;
  for (int32_t e = 0; e < m->n_elems; ++e) {
    const int32_t* t = m->tets10 + 10 * (size_t)e;
    for (int q = 0; q < 6; ++q) {
      int32_t a = t[kEdgeEnds[q][0]], b = t[kEdgeEnds[q][1]];
      if (a > b) { const int32_t s = a; a = b; b = s; }
      ends[2 * (size_t)t[4 + q]] = a;
      ends[2 * (size_t)t[4 + q] + 1] = b;
    }
  }
  p->row_ptr = (int32_t*)malloc(sizeof(int32_t) * ((size_t)p->n_fine + 1));
  p->row_ptr[0] = 0;
  for (int32_t fn = 0; fn < p->n_fine; ++fn) p->row_ptr[fn + 1] = p->row_ptr[fn] + (fn < m->vertex_count ? 1 : 2);
  p->cols = (int32_t*)malloc(sizeof(int32_t) * (size_t)p->row_ptr[p->n_fine]);
  p->weights = (double*)malloc(sizeof(double) * (size_t)p->row_ptr[p->n_fine]);
  for (int32_t fn = 0; fn < p->n_fine; ++fn) {
    const int32_t s = p->row_ptr[fn];
    if (fn < m->vertex_count) {
      p->cols[s] = fn;
      p->weights[s] = 1.0;
    } else {
      if (ends[2 * (size_t)fn] < 0) {
        free(ends);
        return fail(E_VALID, "geometric prolongation: edge node %d not present in edge map", fn);
      }
      p->cols[s] = ends[2 * (size_t)fn];
      p->cols[s + 1] = ends[2 * (size_t)fn + 1];
      p->weights[s] = 0.5;
      p->weights[s + 1] = 0.5;
    }
  }
  free(ends);
  return 0;
}
int or_geo_prolong(const or_mesh* m, int32_t transpose, const float* in, float* out,
                   int32_t batch) {
  or_prolong p;
  const int rc = build_geo(m, &p);
  if (rc) return rc;
  if (transpose) prolong_restrict(&p, in, out, batch);
  else prolong_apply(&p, in, out, batch);
  prolong_free(&p);
  return 0;
}

/* ---------------------------------------------------------- aggregation.hpp */
typedef struct { int32_t* agg_of_node; int32_t n_aggregates; } or_agg;
/* aggregate_p1 (aggregation.hpp:23-89) */
static int aggregate_p1(const or_bcsr* a, int32_t target, or_agg* out) {
  if (target < 2) return fail(E_VALID, "aggregate_p1: target_size must be >= 2");
  const int32_t n = a->n;
  int32_t* agg = (int32_t*)malloc(sizeof(int32_t) * ((size_t)n + 1));
  for (int32_t i = 0; i < n; ++i) agg[i] = -1;
  /* members as a flat list per aggregate: aggregates never exceed target
   * before merging; merges append singletons, so track with linked lists */
  int32_t* msize = (int32_t*)malloc(sizeof(int32_t) * ((size_t)n + 1));
  int32_t* first = (int32_t*)malloc(sizeof(int32_t) * ((size_t)n + 1));  /* first member (for singletons) */
  int32_t* seeds = (int32_t*)malloc(sizeof(int32_t) * ((size_t)n + 1));
  int32_t* queue = (int32_t*)malloc(sizeof(int32_t) * ((size_t)n + 1));
  int32_t nagg = 0;
  for (int32_t seed = 0; seed < n; ++seed) {
    if (agg[seed] >= 0) continue;
    const int32_t id = nagg++;
    msize[id] = 1;
    first[id] = seed;
    seeds[id] = seed;
    agg[seed] = id;
    int32_t qh = 0, qt = 0;
    queue[qt++] = seed;
    while (qh < qt && msize[id] < target) {
      const int32_t node = queue[qh++];
      for (int32_t e = a->row_ptr[node]; e < a->row_ptr[node + 1] && msize[id] < target; ++e) {
        const int32_t nb = a->col_idx[e];
        if (nb == node || agg[nb] >= 0) continue;
        agg[nb] = id;
        ++msize[id];
        queue[qt++] = nb;
      }
    }
  }
  /* singleton merge (aggregation.hpp:55-77) */
  int32_t* remap = (int32_t*)malloc(sizeof(int32_t) * ((size_t)nagg + 1));
  for (int32_t id = 0; id < nagg; ++id) remap[id] = id;
  for (int32_t id = 0; id < nagg; ++id) {
    if (msize[id] != 1) continue;
    const int32_t node = first[id];
    int32_t tgt = -1;
    for (int32_t e = a->row_ptr[node]; e < a->row_ptr[node + 1]; ++e) {
      const int32_t nb = a->col_idx[e];
      if (nb == node) continue;
      const int32_t other = agg[nb];
      if (other != id && msize[remap[other]] > 0) {
        tgt = remap[other];
        break;
      }
    }
    if (tgt >= 0) {
      ++msize[tgt];
      agg[node] = tgt;
      remap[id] = tgt;
      msize[id] = 0;
    }
  }
  /* compact ids preserving creation order (aggregation.hpp:80-87) */
  int32_t* compact = (int32_t*)malloc(sizeof(int32_t) * ((size_t)nagg + 1));
  int32_t na = 0;
  for (int32_t id = 0; id < nagg; ++id) compact[id] = msize[id] > 0 ? na++ : -1;
  for (int32_t node = 0; node < n; ++node) agg[node] = compact[agg[node]];
  out->agg_of_node = agg;
  out->n_aggregates = na;
  free(msize); free(first); free(seeds); free(queue); free(remap); free(compact);
  return 0;
}
/* build_level2 (aggregation.hpp:95-170): P2 and A2 = P^T K1 P (masked fine dofs dropped) */
static int build_level2(const or_bcsr* k1, const or_agg* agg, const uint8_t* fine_mask,
                        or_prolong* p, or_bcsr* a2) {
  const int32_t nf = k1->n, nc = agg->n_aggregates;
  if (nc < 1) return fail(E_VALID, "build_level2: empty aggregation");
  p->n_fine = nf;
  p->n_coarse = nc;
  p->row_ptr = (int32_t*)malloc(sizeof(int32_t) * ((size_t)nf + 1));
  p->cols = (int32_t*)malloc(sizeof(int32_t) * ((size_t)nf + 1));
  p->weights = (double*)malloc(sizeof(double) * ((size_t)nf + 1));
  for (int32_t fn = 0; fn < nf; ++fn) {
    p->row_ptr[fn] = fn;
    p->cols[fn] = agg->agg_of_node[fn];
    p->weights[fn] = 1.0;
  }
  p->row_ptr[nf] = nf;
  /* coarse pattern (:123-139) */
  int32_t* cnt = (int32_t*)calloc((size_t)nc + 1, sizeof(int32_t));
  for (int32_t r = 0; r < nf; ++r) cnt[agg->agg_of_node[r] + 1] += k1->row_ptr[r + 1] - k1->row_ptr[r];
  for (int32_t i = 0; i < nc; ++i) cnt[i + 1] += cnt[i];
  int32_t* buf = (int32_t*)malloc(sizeof(int32_t) * ((size_t)cnt[nc] + 1));
  int32_t* cur = (int32_t*)malloc(sizeof(int32_t) * ((size_t)nc + 1));
  memcpy(cur, cnt, sizeof(int32_t) * (size_t)nc);
  for (int32_t r = 0; r < nf; ++r)
    for (int32_t e = k1->row_ptr[r]; e < k1->row_ptr[r + 1]; ++e)
      buf[cur[agg->agg_of_node[r]]++] = agg->agg_of_node[k1->col_idx[e]];
  a2->n = nc;
  a2->row_ptr = (int32_t*)calloc((size_t)nc + 1, sizeof(int32_t));
  int32_t w = 0;
  for (int32_t r = 0; r < nc; ++r) {
    int32_t* row = buf + cnt[r];
    const int32_t len = cnt[r + 1] - cnt[r];
    qsort(row, (size_t)len, sizeof(int32_t), cmp_i32);
    int32_t u = 0;
    for (int32_t i = 0; i < len; ++i)
      if (u == 0 || row[i] != row[u - 1]) row[u++] = row[i];
    for (int32_t i = 0; i < u; ++i) buf[w + i] = row[i];
    w += u;
    a2->row_ptr[r + 1] = w;
  }
  a2->col_idx = (int32_t*)malloc(sizeof(int32_t) * ((size_t)w + 1));
  memcpy(a2->col_idx, buf, sizeof(int32_t) * (size_t)w);
  free(buf); free(cur); free(cnt);
  a2->blocks = (double*)calloc((size_t)w * 9 + 1, sizeof(double));
  for (int32_t r = 0; r < nf; ++r) {
    const int32_t cr = agg->agg_of_node[r];
    for (int32_t e = k1->row_ptr[r]; e < k1->row_ptr[r + 1]; ++e) {
      const int32_t c = k1->col_idx[e];
      double* dst = a2->blocks + 9 * (size_t)entry_of(a2, cr, agg->agg_of_node[c]);
      const double* src = k1->blocks + 9 * (size_t)e;
      for (int i = 0; i < 3; ++i) {
        if (fine_mask && fine_mask[3 * (size_t)r + i]) continue;
        for (int j = 0; j < 3; ++j) {
          if (fine_mask && fine_mask[3 * (size_t)c + j]) continue;
          dst[3 * i + j] += src[3 * i + j];
        }
      }
    }
  }
  for (int32_t r = 0; r < nc; ++r) {  /* (:164-168) */
    double* d = a2->blocks + 9 * (size_t)entry_of(a2, r, r);
    for (int i = 0; i < 3; ++i)
      if (d[4 * i] == 0.0) d[4 * i] = 1.0;
  }
  return 0;
}

/* ----------------------------------------------------------- vector_batch.hpp */
/* dot_columns (vector_batch.hpp:52-64): sequential fp64 accumulation */
static void dot_f(const float* x, const float* y, int64_t nd, int32_t nb, double* out) {
  for (int32_t b = 0; b < nb; ++b) out[b] = 0.0;
  for (int64_t d = 0; d < nd; ++d)
    for (int32_t b = 0; b < nb; ++b) out[b] += (double)x[d * nb + b] * (double)y[d * nb + b];
}
static void dot_d(const double* x, const double* y, int64_t nd, int32_t nb, double* out) {
  for (int32_t b = 0; b < nb; ++b) out[b] = 0.0;
  for (int64_t d = 0; d < nd; ++d)
    for (int32_t b = 0; b < nb; ++b) out[b] += x[d * nb + b] * y[d * nb + b];
}
/* axpy_columns (:72-83): y += (T)alpha * x */
static void axpy_f(const double* alpha, const float* x, float* y, int64_t nd, int32_t nb) {
  for (int64_t d = 0; d < nd; ++d)
    for (int32_t b = 0; b < nb; ++b) y[d * nb + b] += (float)alpha[b] * x[d * nb + b];
}
static void axpy_d(const double* alpha, const double* x, double* y, int64_t nd, int32_t nb) {
  for (int64_t d = 0; d < nd; ++d)
    for (int32_t b = 0; b < nb; ++b) y[d * nb + b] += alpha[b] * x[d * nb + b];
}
/* xpby_columns (:86-97): p = z + (T)beta * p */
static void xpby_f(const float* z, const double* beta, float* p, int64_t nd, int32_t nb) {
  for (int64_t d = 0; d < nd; ++d)
    for (int32_t b = 0; b < nb; ++b) p[d * nb + b] = z[d * nb + b] + (float)beta[b] * p[d * nb + b];
}
static void xpby_d(const double* z, const double* beta, double* p, int64_t nd, int32_t nb) {
  for (int64_t d = 0; d < nd; ++d)
    for (int32_t b = 0; b < nb; ++b) p[d * nb + b] = z[d * nb + b] + beta[b] * p[d * nb + b];
}
/* zero_masked (:109-119) */
static void zero_masked_f(float* x, const uint8_t* mask, int64_t nd, int32_t nb) {
  if (!mask) return;
  for (int64_t d = 0; d < nd; ++d)
    if (mask[d])
      for (int32_t b = 0; b < nb; ++b) x[d * nb + b] = 0.0f;
}
/* max_rel_ratio (pcg.hpp:32-42) */
static double max_rel_ratio(const double* num2, const double* den2, int32_t nb) {
  double worst = 0.0;
  for (int32_t b = 0; b < nb; ++b) {
    if (den2[b] == 0.0) {
      if (num2[b] != 0.0) return INFINITY;
      continue;
    }
    const double q = num2[b] / den2[b];
    if (q > worst) worst = q;
  }
  return worst;
}

/* --------------------------------------------------------------- pcg.hpp */
typedef struct {
  int kind;              /* 0 = EBE<float>, 1 = BCSR<float> */
  const or_ebe* ebe;
  const or_bcsr* bcsr;   /* float values stored as double */
  int32_t n;
} or_op;
static void op_apply(const or_op* a, const float* u, float* f, int32_t nb) {
  if (a->kind == 0) ebe_apply(a->ebe, u, f, nb);
  else bcsr_apply_t(a->bcsr->n, a->bcsr->row_ptr, a->bcsr->col_idx, a->bcsr->blocks, 32, u, f, nb);
}
typedef struct { float *e, *z, *p, *q; } or_pcgwork;

/* inner_pcg (pcg.hpp:52-124) in 32-bit; bj holds double(float) inverse blocks */
static int inner_pcg(const or_op* a, const double* bj, const float* r, float* u, int32_t nb,
                     double tol, int max_iter, or_pcgwork* w, int* iters, int* converged) {
  if (max_iter < 1) return fail(E_VALID, "inner_pcg: max_iter must be >= 1");
  const int64_t nd = 3 * (int64_t)a->n, len = nd * nb;
  op_apply(a, u, w->e, nb);                                   /* e = r - A u */
  for (int64_t i = 0; i < len; ++i) w->e[i] = r[i] - w->e[i];
  double* rn = (double*)malloc(sizeof(double) * 8 * (size_t)nb);
  double *en = rn + nb, *rho_a = en + nb, *rho_b = rho_a + nb, *beta = rho_b + nb,
         *gamma = beta + nb, *alpha = gamma + nb, *nalpha = alpha + nb;
  for (int32_t b = 0; b < nb; ++b) rho_a[b] = rho_b[b] = beta[b] = gamma[b] = alpha[b] = 0.0;
  dot_f(r, r, nd, nb, rn);
  dot_f(w->e, w->e, nd, nb, en);
  int it = 0;
  const double tol2 = tol * tol;
  double ratio = max_rel_ratio(en, rn, nb);
  int rc = 0;
  if (isnan(ratio)) { rc = fail(E_SOLVER, "inner_pcg: non-finite initial residual"); goto out; }
  while (ratio > tol2 && it < max_iter) {
    bj_apply_t(a->n, bj, 32, w->e, w->z, nb);
    dot_f(w->z, w->e, nd, nb, rho_a);
    if (it == 0) {
      for (int32_t b = 0; b < nb; ++b) beta[b] = 0.0;
      memcpy(w->p, w->z, sizeof(float) * (size_t)len);
    } else {
      for (int32_t b = 0; b < nb; ++b) beta[b] = rho_b[b] != 0.0 ? rho_a[b] / rho_b[b] : 0.0;
      xpby_f(w->z, beta, w->p, nd, nb);
    }
    op_apply(a, w->p, w->q, nb);
    dot_f(w->p, w->q, nd, nb, gamma);
    int stagnated = 0;
    for (int32_t b = 0; b < nb; ++b) {
      if (gamma[b] > 0.0) { alpha[b] = rho_a[b] / gamma[b]; continue; }
      if (gamma[b] == 0.0 && rho_a[b] == 0.0) { alpha[b] = 0.0; continue; }
      double* pn = (double*)malloc(sizeof(double) * 2 * (size_t)nb);
      dot_f(w->p, w->p, nd, nb, pn);
      dot_f(w->q, w->q, nd, nb, pn + nb);
      const double scale = sqrt(pn[b]) * sqrt(pn[nb + b]);
      free(pn);
      const double eps16 = 16.0 * (double)FLT_EPSILON;
      if (fabs(gamma[b]) <= eps16 * scale) { alpha[b] = 0.0; stagnated = 1; continue; }
      rc = fail(E_SOLVER, "inner_pcg: breakdown (p,Ap) <= 0 at iteration %d, column %d", it + 1, b);
      goto out;
    }
    if (stagnated) break;
    for (int32_t b = 0; b < nb; ++b) { rho_b[b] = rho_a[b]; nalpha[b] = -alpha[b]; }
    axpy_f(nalpha, w->q, w->e, nd, nb);
    axpy_f(alpha, w->p, u, nd, nb);
    ++it;
    dot_f(w->e, w->e, nd, nb, en);
    ratio = max_rel_ratio(en, rn, nb);
    if (isnan(ratio)) { rc = fail(E_SOLVER, "inner_pcg: non-finite residual at iteration %d", it); goto out; }
  }
out:
  *iters = it;
  *converged = ratio <= tol2;
  free(rn);
  return rc;
}
static void work_alloc(or_pcgwork* w, size_t len) {
  w->e = (float*)calloc(len + 1, sizeof(float));
  w->z = (float*)calloc(len + 1, sizeof(float));
  w->p = (float*)calloc(len + 1, sizeof(float));
  w->q = (float*)calloc(len + 1, sizeof(float));
}
static void work_free(or_pcgwork* w) { free(w->e); free(w->z); free(w->p); free(w->q); }

int or_inner_pcg_ebe(const or_mesh* m, int32_t order, int32_t n_mat, const double* lam,
                     const double* mu, const uint8_t* mask, const float* r, float* u,
                     int32_t batch, double tol, int32_t max_iter, int32_t* iters,
                     int32_t* converged) {
  or_ebe op;
  memset(&op, 0, sizeof op);
  int rc = ebe_init(&op, m, order, n_mat, lam, mu, mask, 32);
  if (rc) { ebe_free(&op); return rc; }
  double* bj = (double*)malloc(sizeof(double) * 9 * (size_t)op.n_nodes);
  rc = ebe_bj(&op, bj);
  if (rc == 0) {
    or_op a = {0, &op, NULL, op.n_nodes};
    or_pcgwork w;
    work_alloc(&w, (size_t)3 * op.n_nodes * batch);
    int it = 0, cv = 0;
    rc = inner_pcg(&a, bj, r, u, batch, tol, max_iter, &w, &it, &cv);
    *iters = it;
    *converged = cv;
    work_free(&w);
  }
  free(bj);
  ebe_free(&op);
  return rc;
}

/* --------------------------------------------------------- adaptive_cg.hpp */
typedef struct {
  or_ebe outer, level0, level1;
  or_bcsr level2;          /* float values stored as double */
  or_prolong p1, p2;
  double *m0, *m1, *m2;    /* inverse blocks, double(float) */
  uint8_t *mask0, *mask1, *mask2;
  or_agg agg;
} or_levels;

static int validate_cfg(const ts_solver_config* c) {
  const double t[4] = {c->outer_tol, c->level_tol[0], c->level_tol[1], c->level_tol[2]};
  for (int i = 0; i < 4; ++i)
    if (!(t[i] > 0.0 && t[i] < 1.0)) return fail(E_VALID, "solver config: tolerance must lie in (0, 1)");
  if (c->outer_max_iter < 1 || c->level_max_iter[0] < 1 || c->level_max_iter[1] < 1 || c->level_max_iter[2] < 1)
    return fail(E_VALID, "solver config: max iterations must be >= 1");
  if (c->batch_size < 1) return fail(E_VALID, "solver config: batch size must be >= 1");
  if (c->aggregate_target < 2) return fail(E_VALID, "solver config: aggregate target must be >= 2");
  return 0;
}

/* build_solver_levels (adaptive_cg.hpp:39-67) on dirichlet_mask(mesh) (model.hpp:21-29) */
void* or_levels_create(const or_mesh* m, int32_t n_mat, const double* lam, const double* mu,
                       const ts_solver_config* cfg, int32_t workers, double* setup_s) {
  (void)workers;
  const double t0 = now_s();
  if (validate_cfg(cfg)) return NULL;
  or_levels* lv = (or_levels*)calloc(1, sizeof(or_levels));
  const size_t nn = (size_t)m->n_nodes, nv = (size_t)m->vertex_count;
  lv->mask0 = (uint8_t*)malloc(3 * nn);
  or_mesh_mask(m, lv->mask0);
  lv->mask1 = (uint8_t*)malloc(3 * nv + 1);
  memcpy(lv->mask1, lv->mask0, 3 * nv);
  if (ebe_init(&lv->outer, m, 2, n_mat, lam, mu, lv->mask0, 64) ||
      ebe_init(&lv->level0, m, 2, n_mat, lam, mu, lv->mask0, 32) ||
      ebe_init(&lv->level1, m, 1, n_mat, lam, mu, lv->mask1, 32) || build_geo(m, &lv->p1)) {
    or_levels_destroy(lv);
    return NULL;
  }
  or_ebe k1d;
  memset(&k1d, 0, sizeof k1d);
  ebe_init(&k1d, m, 1, n_mat, lam, mu, lv->mask1, 64);
  or_bcsr* k1 = assemble(&k1d);
  ebe_free(&k1d);
  if (aggregate_p1(k1, cfg->aggregate_target, &lv->agg) ||
      build_level2(k1, &lv->agg, lv->mask1, &lv->p2, &lv->level2)) {
    or_bcsr_destroy(k1);
    or_levels_destroy(lv);
    return NULL;
  }
  or_bcsr_destroy(k1);
  const size_t nb2 = (size_t)lv->level2.row_ptr[lv->level2.n];
  for (size_t q = 0; q < 9 * nb2; ++q) lv->level2.blocks[q] = (double)(float)lv->level2.blocks[q]; /* cast_bcsr<float> */
  /* coarse_mask (aggregation.hpp:174-185) */
  const int32_t n2 = lv->agg.n_aggregates;
  lv->mask2 = (uint8_t*)malloc(3 * (size_t)n2 + 1);
  memset(lv->mask2, 1, 3 * (size_t)n2);
  for (size_t node = 0; node < nv; ++node)
    for (int i = 0; i < 3; ++i)
      if (!lv->mask1[3 * node + i]) lv->mask2[3 * (size_t)lv->agg.agg_of_node[node] + i] = 0;
  lv->m0 = (double*)malloc(sizeof(double) * 9 * nn);
  lv->m1 = (double*)malloc(sizeof(double) * 9 * nv);
  lv->m2 = (double*)malloc(sizeof(double) * 9 * (size_t)n2);
  if (ebe_bj(&lv->level0, lv->m0) || ebe_bj(&lv->level1, lv->m1) || bcsr_bj(&lv->level2, 32, lv->m2)) {
    or_levels_destroy(lv);
    return NULL;
  }
  if (setup_s) *setup_s = now_s() - t0;
  return lv;
}
void or_levels_sizes(const void* h, int32_t* n0, int32_t* n1, int32_t* n2, int64_t* nnzb2) {
  const or_levels* lv = (const or_levels*)h;
  *n0 = lv->level0.n_nodes;
  *n1 = lv->level1.n_nodes;
  *n2 = lv->level2.n;
  *nnzb2 = lv->level2.row_ptr[lv->level2.n];
}
void or_levels_export(const void* h, int32_t* agg, int32_t* row_ptr2, int32_t* col_idx2,
                      float* blocks2, uint8_t* mask2, float* m0, float* m1, float* m2) {
  const or_levels* lv = (const or_levels*)h;
  const int32_t n2 = lv->level2.n;
  const int64_t nb2 = lv->level2.row_ptr[n2];
  if (agg) memcpy(agg, lv->agg.agg_of_node, sizeof(int32_t) * (size_t)lv->level1.n_nodes);
  if (row_ptr2) memcpy(row_ptr2, lv->level2.row_ptr, sizeof(int32_t) * ((size_t)n2 + 1));
  if (col_idx2) memcpy(col_idx2, lv->level2.col_idx, sizeof(int32_t) * (size_t)nb2);
  if (blocks2) for (int64_t q = 0; q < 9 * nb2; ++q) blocks2[q] = (float)lv->level2.blocks[q];
  if (mask2) memcpy(mask2, lv->mask2, 3 * (size_t)n2);
  if (m0) for (size_t q = 0; q < 9 * (size_t)lv->level0.n_nodes; ++q) m0[q] = (float)lv->m0[q];
  if (m1) for (size_t q = 0; q < 9 * (size_t)lv->level1.n_nodes; ++q) m1[q] = (float)lv->m1[q];
  if (m2) for (size_t q = 0; q < 9 * (size_t)n2; ++q) m2[q] = (float)lv->m2[q];
}
void or_levels_destroy(void* h) {
  or_levels* lv = (or_levels*)h;
  if (!lv) return;
  ebe_free(&lv->outer); ebe_free(&lv->level0); ebe_free(&lv->level1);
  bcsr_free(&lv->level2);
  prolong_free(&lv->p1); prolong_free(&lv->p2);
  free(lv->m0); free(lv->m1); free(lv->m2);
  free(lv->mask0); free(lv->mask1); free(lv->mask2);
  free(lv->agg.agg_of_node);
  free(lv);
}
int or_levels_outer_apply(const void* h, const double* u, double* f, int32_t batch) {
  ebe_apply(&((const or_levels*)h)->outer, u, f, batch);
  return 0;
}

typedef struct {
  float *r0, *u0, *r1, *u1, *r2, *u2;
  or_pcgwork w0, w1, w2;
} or_mcycle;

/* apply_multigrid_preconditioner (adaptive_cg.hpp:80-120) */
static int mg_precond(const or_levels* lv, const ts_solver_config* cfg, const double* r,
                      double* z, int32_t nb, or_mcycle* w, ts_solve_report* rep) {
  const int64_t n0 = 3 * (int64_t)lv->level0.n_nodes * nb, n1d = 3 * (int64_t)lv->level1.n_nodes,
                n2d = 3 * (int64_t)lv->level2.n;
  for (int64_t i = 0; i < n0; ++i) w->r0[i] = (float)r[i];        /* cast_batch */
  bj_apply_t(lv->level0.n_nodes, lv->m0, 32, w->r0, w->u0, nb);
  prolong_restrict(&lv->p1, w->r0, w->r1, nb);
  prolong_restrict(&lv->p1, w->u0, w->u1, nb);
  zero_masked_f(w->r1, lv->mask1, n1d, nb);
  zero_masked_f(w->u1, lv->mask1, n1d, nb);
  prolong_restrict(&lv->p2, w->r1, w->r2, nb);
  prolong_restrict(&lv->p2, w->u1, w->u2, nb);
  zero_masked_f(w->r2, lv->mask2, n2d, nb);
  zero_masked_f(w->u2, lv->mask2, n2d, nb);
  int it2, it1, it0, cv, rc;
  double t0 = now_s();
  or_op a2 = {1, NULL, &lv->level2, lv->level2.n};
  rc = inner_pcg(&a2, lv->m2, w->r2, w->u2, nb, cfg->level_tol[2], cfg->level_max_iter[2], &w->w2, &it2, &cv);
  if (rc) return rc;
  double t1 = now_s();
  prolong_apply(&lv->p2, w->u2, w->u1, nb);
  zero_masked_f(w->u1, lv->mask1, n1d, nb);
  or_op a1 = {0, &lv->level1, NULL, lv->level1.n_nodes};
  rc = inner_pcg(&a1, lv->m1, w->r1, w->u1, nb, cfg->level_tol[1], cfg->level_max_iter[1], &w->w1, &it1, &cv);
  if (rc) return rc;
  double t2 = now_s();
  prolong_apply(&lv->p1, w->u1, w->u0, nb);
  zero_masked_f(w->u0, lv->mask0, 3 * (int64_t)lv->level0.n_nodes, nb);
  or_op a0 = {0, &lv->level0, NULL, lv->level0.n_nodes};
  rc = inner_pcg(&a0, lv->m0, w->r0, w->u0, nb, cfg->level_tol[0], cfg->level_max_iter[0], &w->w0, &it0, &cv);
  if (rc) return rc;
  double t3 = now_s();
  rep->inner_iterations[2] += it2;
  rep->inner_iterations[1] += it1;
  rep->inner_iterations[0] += it0;
  rep->time_inner_s[2] += t1 - t0;
  rep->time_inner_s[1] += t2 - t1;
  rep->time_inner_s[0] += t3 - t2;
  for (int64_t i = 0; i < n0; ++i) z[i] = (double)w->u0[i];
  return 0;
}

typedef int (*precond_fn)(void* ctx, const double* r, double* z);

/* run_outer_cg (adaptive_cg.hpp:126-233) */
static int run_outer_cg(const or_ebe* k, const double* f, double* u, int32_t nb, double tol,
                        int max_iter, int hist_stride, precond_fn precond, void* ctx,
                        ts_solve_report* rep) {
  const double t_start = now_s();
  const int64_t nd = 3 * (int64_t)k->n_nodes, len = nd * nb;
  double* fn2 = (double*)malloc(sizeof(double) * 9 * (size_t)nb);
  double *rn2 = fn2 + nb, *rho = rn2 + nb, *gprev = rho + nb, *beta = gprev + nb, *alpha = beta + nb,
         *gamma = alpha + nb, *nalpha = gamma + nb, *zq = nalpha + nb;
  for (int32_t b = 0; b < nb; ++b) gprev[b] = beta[b] = 0.0;
  dot_d(f, f, nd, nb, fn2);
  double* r = (double*)calloc((size_t)len + 1, sizeof(double));
  double* q = (double*)calloc((size_t)len + 1, sizeof(double));
  double* z = (double*)calloc((size_t)len + 1, sizeof(double));
  double* p = (double*)calloc((size_t)len + 1, sizeof(double));
  double* scratch = (double*)calloc((size_t)len + 1, sizeof(double));
  int rc = 0;
#define TRUE_RESIDUAL()                                          \
  do {                                                           \
    ebe_apply(k, u, scratch, nb);                                \
    for (int64_t i = 0; i < len; ++i) r[i] = f[i] - scratch[i];  \
    dot_d(r, r, nd, nb, rn2);                                    \
  } while (0)
  TRUE_RESIDUAL();
  const double tol2 = tol * tol;
  rep->batch_size = nb;
  int it = 0, r_is_true = 1, first = 1;
  while (1) {
    double ratio = max_rel_ratio(rn2, fn2, nb);
    if (isnan(ratio)) { rc = fail(E_SOLVER, "solve: non-finite residual"); goto done; }
    if (ratio <= tol2) {
      if (r_is_true) break;
      TRUE_RESIDUAL();
      r_is_true = 1;
      ratio = max_rel_ratio(rn2, fn2, nb);
      if (ratio <= tol2) break;
    }
    if (it >= max_iter) {
      if (!r_is_true) TRUE_RESIDUAL();
      rep->outer_iterations = it;
      rep->converged = 0;
      rc = fail(E_CONV, "solve: outer loop did not converge within %d iterations (max residual %f)", max_iter, sqrt(ratio));
      goto done;
    }
    rc = precond(ctx, r, z);
    if (rc) goto done;
    if (first) {
      for (int32_t b = 0; b < nb; ++b) beta[b] = 0.0;
      memcpy(p, z, sizeof(double) * (size_t)len);
      first = 0;
    } else {
      dot_d(z, q, nd, nb, zq);
      for (int32_t b = 0; b < nb; ++b) beta[b] = gprev[b] != 0.0 ? -zq[b] / gprev[b] : 0.0;
      xpby_d(z, beta, p, nd, nb);
    }
    ebe_apply(k, p, q, nb);
    dot_d(z, r, nd, nb, rho);
    dot_d(p, q, nd, nb, gamma);
    for (int32_t b = 0; b < nb; ++b) {
      if (gamma[b] > 0.0) alpha[b] = rho[b] / gamma[b];
      else if (gamma[b] == 0.0 && rho[b] == 0.0) alpha[b] = 0.0;
      else { rc = fail(E_SOLVER, "solve: breakdown (p,Kp) <= 0 at outer iteration %d, column %d", it + 1, b); goto done; }
      nalpha[b] = -alpha[b];
    }
    for (int32_t b = 0; b < nb; ++b) gprev[b] = gamma[b];
    axpy_d(nalpha, q, r, nd, nb);
    axpy_d(alpha, p, u, nd, nb);
    r_is_true = 0;
    ++it;
    dot_d(r, r, nd, nb, rn2);
    if (hist_stride > 0 && it % hist_stride == 0 && rep->history_count < rep->history_capacity) {
      const int32_t row = rep->history_count;
      if (rep->history_iter) rep->history_iter[row] = it;
      if (rep->history)
        for (int32_t b = 0; b < nb; ++b)
          rep->history[(size_t)row * nb + b] = fn2[b] > 0.0 ? sqrt(rn2[b] / fn2[b]) : 0.0;
      rep->history_count++;
    }
  }
  rep->outer_iterations = it;
  rep->converged = 1;
done:
  /* finalize (:150-160) */
  if (rep->final_rel_residual)
    for (int32_t b = 0; b < nb; ++b)
      rep->final_rel_residual[b] = fn2[b] > 0.0 ? sqrt(rn2[b] / fn2[b]) : (rn2[b] > 0.0 ? INFINITY : 0.0);
  rep->time_total_s = now_s() - t_start;
  rep->time_outer_s = rep->time_total_s - rep->time_inner_s[0] - rep->time_inner_s[1] - rep->time_inner_s[2];
#undef TRUE_RESIDUAL
  free(fn2); free(r); free(q); free(z); free(p); free(scratch);
  return rc;
}

typedef struct { const or_levels* lv; const ts_solver_config* cfg; or_mcycle w; ts_solve_report* rep; int32_t nb; } mg_ctx;
static int mg_cb(void* c, const double* r, double* z) {
  mg_ctx* m = (mg_ctx*)c;
  return mg_precond(m->lv, m->cfg, r, z, m->nb, &m->w, m->rep);
}
static void report_init(ts_solve_report* rep, int method, int prec) {
  rep->converged = 0;
  rep->outer_iterations = 0;
  for (int i = 0; i < 3; ++i) { rep->inner_iterations[i] = 0; rep->time_inner_s[i] = 0.0; }
  rep->time_setup_s = rep->time_outer_s = rep->time_total_s = 0.0;
  rep->history_count = 0;
  rep->method = method;
  rep->inner_precision = prec;
}

/* solve (adaptive_cg.hpp:242-263) */
int or_solve(const void* h, const double* f, const double* u0, double* u_out, int32_t batch,
             const ts_solver_config* cfg, ts_solve_report* rep) {
  const or_levels* lv = (const or_levels*)h;
  int rc = validate_cfg(cfg);
  if (rc) return rc;
  const int64_t nd = 3 * (int64_t)lv->outer.n_nodes, len = nd * batch;
  double* fn2 = (double*)malloc(sizeof(double) * (size_t)batch);
  dot_d(f, f, nd, batch, fn2);
  int any = 0;
  for (int32_t b = 0; b < batch; ++b) any |= fn2[b] != 0.0;
  free(fn2);
  if (!any) return fail(E_VALID, "solve: right-hand side has no nonzero column");
  report_init(rep, 0, 32);
  rep->batch_size = batch;
  if (u_out != u0) memcpy(u_out, u0, sizeof(double) * (size_t)len);
  mg_ctx c;
  c.lv = lv; c.cfg = cfg; c.rep = rep; c.nb = batch;
  const size_t l0 = (size_t)3 * lv->level0.n_nodes * batch, l1 = (size_t)3 * lv->level1.n_nodes * batch,
               l2 = (size_t)3 * lv->level2.n * batch;
  c.w.r0 = (float*)calloc(l0 + 1, 4); c.w.u0 = (float*)calloc(l0 + 1, 4);
  c.w.r1 = (float*)calloc(l1 + 1, 4); c.w.u1 = (float*)calloc(l1 + 1, 4);
  c.w.r2 = (float*)calloc(l2 + 1, 4); c.w.u2 = (float*)calloc(l2 + 1, 4);
  work_alloc(&c.w.w0, l0); work_alloc(&c.w.w1, l1); work_alloc(&c.w.w2, l2);
  rc = run_outer_cg(&lv->outer, f, u_out, batch, cfg->outer_tol, cfg->outer_max_iter,
                    cfg->residual_history_stride, mg_cb, &c, rep);
  free(c.w.r0); free(c.w.u0); free(c.w.r1); free(c.w.u1); free(c.w.r2); free(c.w.u2);
  work_free(&c.w.w0); work_free(&c.w.w1); work_free(&c.w.w2);
  return rc;
}

typedef struct { const double* m; int32_t n, nb; } bj_ctx;
static int bj_cb(void* c, const double* r, double* z) {
  bj_ctx* b = (bj_ctx*)c;
  bj_apply_t(b->n, b->m, 64, r, z, b->nb);
  return 0;
}
/* solve_pcge (adaptive_cg.hpp:267-279): outer CG with the 64-bit block Jacobi;
 * residual history at stride 0 (the reference's SolveReport default) */
int or_solve_pcge(const void* h, const double* f, const double* u0, double* u_out,
                  int32_t batch, double tol, int32_t max_iter, ts_solve_report* rep) {
  const or_levels* lv = (const or_levels*)h;
  report_init(rep, 1, 64);
  const int64_t len = 3 * (int64_t)lv->outer.n_nodes * batch;
  double* m = (double*)malloc(sizeof(double) * 9 * (size_t)lv->outer.n_nodes);
  int rc = ebe_bj(&lv->outer, m);
  if (rc) { free(m); return rc; }
  if (u_out != u0) memcpy(u_out, u0, sizeof(double) * (size_t)len);
  bj_ctx c = {m, lv->outer.n_nodes, batch};
  rc = run_outer_cg(&lv->outer, f, u_out, batch, tol, max_iter, 0, bj_cb, &c, rep);
  free(m);
  return rc;
}
