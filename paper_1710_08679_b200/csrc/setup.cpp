// setup.cpp — host-side construction of the multigrid hierarchy that the
// device solver runs on (build_solver_levels, adaptive_cg.hpp:39-67).
//
// Level 2 is defined by the reference's SEQUENTIAL greedy aggregation
// (aggregate_p1, aggregation.hpp:23-89): ascending seeds, BFS over the block
// graph of the assembled first-order operator K1, singleton merge, compaction
// in creation order. Any other (e.g. parallel) aggregation would change the
// level-2 operator and with it the iteration counts, so it is reproduced
// exactly here. Assembly of K1 and the Galerkin product are O(E) host passes
// (parallel over rows with OpenMP); all per-iteration work runs on the GPU.
#include "setup.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <deque>

namespace tsg {

namespace {

// inverse of a 3x3 (geometry.hpp:38-52 formula); false when |det| <= min_det
bool invert3(const double m[3][3], double inv[3][3], double min_det) {
  const double d = m[0][0] * (m[1][1] * m[2][2] - m[1][2] * m[2][1]) -
                   m[0][1] * (m[1][0] * m[2][2] - m[1][2] * m[2][0]) +
                   m[0][2] * (m[1][0] * m[2][1] - m[1][1] * m[2][0]);
  if (std::abs(d) <= min_det || d == 0.0) return false;
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
  return true;
}

int32_t find_col(const BcsrD& a, int32_t r, int32_t c) {
  const int32_t* lo = a.col_idx.data() + a.row_ptr[r];
  const int32_t* hi = a.col_idx.data() + a.row_ptr[r + 1];
  return static_cast<int32_t>(std::lower_bound(lo, hi, c) - a.col_idx.data());
}

}  // namespace

// assemble_bcsr(EbeOperator<double>(mesh, 1, ...)) (ebe_operator.hpp:230-284)
// for the first-order vertex grid with the level-1 mask. With `blocks32`, the
// same pass also assembles the fp32 operator's image (float-rounded vertices
// and Lame values, as EbeOperator<float> stores them, ebe_operator.hpp:54-62;
// summed in fp64, stored as float) on the same pattern.
BcsrD assemble_tet4(const Mesh& m, const std::vector<double>& lam_e, const std::vector<double>& mu_e,
                    const std::vector<uint8_t>& mask1, HostVec<float>* blocks32) {
  auto r32 = [](double x) { return static_cast<double>(static_cast<float>(x)); };
  const int32_t n = m.vertex_count;
  const int64_t E = m.n_elems();
  // node -> elements CSR: parallel counting sort, then each row's list sorted, so rows keep the
  // ascending element order the reference's assembly sums in
  std::vector<int64_t> nptr(n + 1, 0);
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < E; ++e)
    for (int a = 0; a < 4; ++a) __atomic_fetch_add(&nptr[m.tets10[10 * e + a] + 1], int64_t(1), __ATOMIC_RELAXED);
  for (int32_t i = 0; i < n; ++i) nptr[i + 1] += nptr[i];
  HostVec<int32_t> nel(nptr[n]);
  {
    std::vector<int64_t> cur(nptr.begin(), nptr.end() - 1);
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < E; ++e)
      for (int a = 0; a < 4; ++a)
        nel[__atomic_fetch_add(&cur[m.tets10[10 * e + a]], int64_t(1), __ATOMIC_RELAXED)] = static_cast<int32_t>(e);
#pragma omp parallel for schedule(dynamic, 4096)
    for (int32_t r = 0; r < n; ++r) std::sort(nel.begin() + nptr[r], nel.begin() + nptr[r + 1]);
  }
  setup_mark("assemble: incidence");
  BcsrD A;
  A.n = n;
  A.row_ptr.assign(n + 1, 0);
  // pattern: sorted unique vertex neighbours (incl. self), counted then filled in place
#pragma omp parallel
  {
    std::vector<int32_t> row;
#pragma omp for schedule(dynamic, 4096)
    for (int32_t r = 0; r < n; ++r) {
      row.clear();
      for (int64_t k = nptr[r]; k < nptr[r + 1]; ++k)
        for (int a = 0; a < 4; ++a) row.push_back(m.tets10[10 * int64_t(nel[k]) + a]);
      std::sort(row.begin(), row.end());
      A.row_ptr[r + 1] = static_cast<int32_t>(std::unique(row.begin(), row.end()) - row.begin());
    }
  }
  for (int32_t r = 0; r < n; ++r) A.row_ptr[r + 1] += A.row_ptr[r];
  A.col_idx.resize(A.row_ptr[n]);
#pragma omp parallel
  {
    std::vector<int32_t> row;
#pragma omp for schedule(dynamic, 4096)
    for (int32_t r = 0; r < n; ++r) {
      row.clear();
      for (int64_t k = nptr[r]; k < nptr[r + 1]; ++k)
        for (int a = 0; a < 4; ++a) row.push_back(m.tets10[10 * int64_t(nel[k]) + a]);
      std::sort(row.begin(), row.end());
      std::unique(row.begin(), row.end());
      std::copy(row.begin(), row.begin() + (A.row_ptr[r + 1] - A.row_ptr[r]), A.col_idx.begin() + A.row_ptr[r]);
    }
  }
  setup_mark("assemble: pattern");
  A.blocks.resize(static_cast<size_t>(A.row_ptr[n]) * 9);
  if (blocks32) blocks32->resize(A.blocks.size());
  // values: row-owner accumulation (each row summed by one thread, element order)
  struct Geo {
    double g[4][3], wl, wm;
    bool ok;
  };
  auto geometry = [&](const int32_t* t, int64_t e, bool round) {
    Geo G{};
    double v[4][3];
    for (int a = 0; a < 4; ++a)
      for (int c = 0; c < 3; ++c) {
        const double x = m.coords[3 * size_t(t[a]) + c];
        v[a][c] = round ? r32(x) : x;
      }
    double j[3][3], inv[3][3];
    for (int c = 0; c < 3; ++c)
      for (int q = 0; q < 3; ++q) j[q][c] = v[c + 1][q] - v[0][q];
    G.ok = invert3(j, inv, 0.0);
    if (!G.ok) return G;
    const double det = j[0][0] * (j[1][1] * j[2][2] - j[1][2] * j[2][1]) -
                       j[0][1] * (j[1][0] * j[2][2] - j[1][2] * j[2][0]) +
                       j[0][2] * (j[1][0] * j[2][1] - j[1][1] * j[2][0]);
    const double vol = det / 6.0;
    for (int d = 0; d < 3; ++d) {
      G.g[1][d] = inv[0][d];
      G.g[2][d] = inv[1][d];
      G.g[3][d] = inv[2][d];
      G.g[0][d] = -(G.g[1][d] + G.g[2][d] + G.g[3][d]);
    }
    G.wl = vol * (round ? r32(lam_e[e]) : lam_e[e]);
    G.wm = vol * (round ? r32(mu_e[e]) : mu_e[e]);
    return G;
  };
  auto add = [&](const Geo& G, int a, int b, int32_t r, int32_t gb, double* blk) {
    const double gdot = G.g[a][0] * G.g[b][0] + G.g[a][1] * G.g[b][1] + G.g[a][2] * G.g[b][2];
    for (int i = 0; i < 3; ++i) {
      if (mask1[3 * size_t(r) + i]) continue;
      for (int jj = 0; jj < 3; ++jj) {
        if (mask1[3 * size_t(gb) + jj]) continue;
        blk[3 * i + jj] += G.wl * G.g[a][i] * G.g[b][jj] + G.wm * G.g[b][i] * G.g[a][jj] + (i == jj ? G.wm * gdot : 0.0);
      }
    }
  };
#pragma omp parallel
  {
    std::vector<double> acc32;
#pragma omp for schedule(dynamic, 4096)
    for (int32_t r = 0; r < n; ++r) {
      const int32_t rb = A.row_ptr[r], len = A.row_ptr[r + 1] - rb;
      std::fill(A.blocks.begin() + 9 * size_t(rb), A.blocks.begin() + 9 * size_t(rb + len), 0.0);
      if (blocks32) acc32.assign(9 * size_t(len), 0.0);
      for (int64_t k = nptr[r]; k < nptr[r + 1]; ++k) {
        const int64_t e = nel[k];
        const int32_t* t = m.tets10.data() + 10 * e;
        const Geo G = geometry(t, e, false);
        const Geo G32 = blocks32 ? geometry(t, e, true) : Geo{};
        int a = 0;
        while (t[a] != r) ++a;
        for (int b = 0; b < 4; ++b) {
          const int32_t gb = t[b];
          const int32_t q = find_col(A, r, gb);
          if (G.ok) add(G, a, b, r, gb, A.blocks.data() + 9 * static_cast<size_t>(q));
          if (blocks32 && G32.ok) add(G32, a, b, r, gb, acc32.data() + 9 * static_cast<size_t>(q - rb));
        }
      }
      const int32_t qd = find_col(A, r, r);
      for (int i = 0; i < 3; ++i)
        if (mask1[3 * size_t(r) + i]) {
          A.blocks[9 * static_cast<size_t>(qd) + 4 * i] = 1.0;
          if (blocks32) acc32[9 * static_cast<size_t>(qd - rb) + 4 * i] = 1.0;
        }
      if (blocks32)
        for (size_t x = 0; x < 9 * size_t(len); ++x) (*blocks32)[9 * size_t(rb) + x] = static_cast<float>(acc32[x]);
    }
  }
  return A;
}

// aggregate_p1 (aggregation.hpp:23-89), sequential and order-exact.
Aggregation aggregate_p1(const BcsrD& a, int32_t target) {
  if (target < 2) validation("aggregate_p1: target_size must be >= 2");
  const int32_t n = a.n;
  Aggregation agg;
  agg.agg_of_node.assign(n, -1);
  std::vector<int32_t> msize, first;
  msize.reserve(n / 4 + 16);
  first.reserve(n / 4 + 16);
  std::vector<int32_t> queue(n + 1);
  for (int32_t seed = 0; seed < n; ++seed) {
    if (agg.agg_of_node[seed] >= 0) continue;
    const int32_t id = static_cast<int32_t>(msize.size());
    msize.push_back(1);
    first.push_back(seed);
    agg.agg_of_node[seed] = id;
    int32_t qh = 0, qt = 0;
    queue[qt++] = seed;
    while (qh < qt && msize[id] < target) {
      const int32_t node = queue[qh++];
      for (int32_t e = a.row_ptr[node]; e < a.row_ptr[node + 1] && msize[id] < target; ++e) {
        const int32_t nb = a.col_idx[e];
        if (nb == node || agg.agg_of_node[nb] >= 0) continue;
        agg.agg_of_node[nb] = id;
        ++msize[id];
        queue[qt++] = nb;
      }
    }
  }
  const int32_t nagg = static_cast<int32_t>(msize.size());
  std::vector<int32_t> remap(nagg);
  for (int32_t id = 0; id < nagg; ++id) remap[id] = id;
  for (int32_t id = 0; id < nagg; ++id) {
    if (msize[id] != 1) continue;
    const int32_t node = first[id];
    int32_t target_id = -1;
    for (int32_t e = a.row_ptr[node]; e < a.row_ptr[node + 1]; ++e) {
      const int32_t nb = a.col_idx[e];
      if (nb == node) continue;
      const int32_t other = agg.agg_of_node[nb];
      if (other != id && msize[remap[other]] > 0) {
        target_id = remap[other];
        break;
      }
    }
    if (target_id >= 0) {
      ++msize[target_id];
      agg.agg_of_node[node] = target_id;
      remap[id] = target_id;
      msize[id] = 0;
    }
  }
  std::vector<int32_t> compact(nagg, -1);
  for (int32_t id = 0; id < nagg; ++id)
    if (msize[id] > 0) {
      compact[id] = agg.n_aggregates++;
      agg.seeds.push_back(first[id]);
    }
  for (int32_t node = 0; node < n; ++node) agg.agg_of_node[node] = compact[agg.agg_of_node[node]];
  return agg;
}

// build_level2 (aggregation.hpp:95-170): A2 = P^T K1 P, masked fine dofs dropped,
// zero coarse diagonals -> 1.
BcsrD build_level2(const BcsrD& k1, const Aggregation& agg, const std::vector<uint8_t>& fine_mask) {
  const int32_t nf = k1.n, nc = agg.n_aggregates;
  if (nc < 1) validation("build_level2: empty aggregation");
  // fine nodes per aggregate (ascending)
  std::vector<int32_t> aptr(nc + 1, 0), amem(nf);
  for (int32_t r = 0; r < nf; ++r) ++aptr[agg.agg_of_node[r] + 1];
  for (int32_t i = 0; i < nc; ++i) aptr[i + 1] += aptr[i];
  {
    std::vector<int32_t> cur(aptr.begin(), aptr.end() - 1);
    for (int32_t r = 0; r < nf; ++r) amem[cur[agg.agg_of_node[r]]++] = r;
  }
  BcsrD a2;
  a2.n = nc;
  a2.row_ptr.assign(nc + 1, 0);
  std::vector<std::vector<int32_t>> rows(nc);
#pragma omp parallel for schedule(dynamic, 1024)
  for (int32_t c = 0; c < nc; ++c) {
    auto& row = rows[c];
    for (int32_t q = aptr[c]; q < aptr[c + 1]; ++q) {
      const int32_t r = amem[q];
      for (int32_t e = k1.row_ptr[r]; e < k1.row_ptr[r + 1]; ++e) row.push_back(agg.agg_of_node[k1.col_idx[e]]);
    }
    std::sort(row.begin(), row.end());
    row.erase(std::unique(row.begin(), row.end()), row.end());
  }
  for (int32_t c = 0; c < nc; ++c) a2.row_ptr[c + 1] = a2.row_ptr[c] + static_cast<int32_t>(rows[c].size());
  a2.col_idx.resize(a2.row_ptr[nc]);
  for (int32_t c = 0; c < nc; ++c) std::copy(rows[c].begin(), rows[c].end(), a2.col_idx.begin() + a2.row_ptr[c]);
  a2.blocks.assign(static_cast<size_t>(a2.row_ptr[nc]) * 9, 0.0);
#pragma omp parallel for schedule(dynamic, 1024)
  for (int32_t cr = 0; cr < nc; ++cr) {
    for (int32_t q = aptr[cr]; q < aptr[cr + 1]; ++q) {
      const int32_t r = amem[q];
      for (int32_t e = k1.row_ptr[r]; e < k1.row_ptr[r + 1]; ++e) {
        const int32_t c = k1.col_idx[e];
        double* dst = a2.blocks.data() + 9 * static_cast<size_t>(find_col(a2, cr, agg.agg_of_node[c]));
        const double* src = k1.blocks.data() + 9 * static_cast<size_t>(e);
        for (int i = 0; i < 3; ++i) {
          if (!fine_mask.empty() && fine_mask[3 * size_t(r) + i]) continue;
          for (int j = 0; j < 3; ++j) {
            if (!fine_mask.empty() && fine_mask[3 * size_t(c) + j]) continue;
            dst[3 * i + j] += src[3 * i + j];
          }
        }
      }
    }
    double* d = a2.blocks.data() + 9 * static_cast<size_t>(find_col(a2, cr, cr));
    for (int i = 0; i < 3; ++i)
      if (d[4 * i] == 0.0) d[4 * i] = 1.0;
  }
  return a2;
}

// coarse_mask (aggregation.hpp:174-185)
std::vector<uint8_t> coarse_mask(const Aggregation& agg, const std::vector<uint8_t>& fine_mask) {
  std::vector<uint8_t> out(3 * static_cast<size_t>(agg.n_aggregates), 1);
  if (fine_mask.empty()) {
    std::fill(out.begin(), out.end(), 0);
    return out;
  }
  for (size_t node = 0; node < agg.agg_of_node.size(); ++node)
    for (int i = 0; i < 3; ++i)
      if (!fine_mask[3 * node + i]) out[3 * static_cast<size_t>(agg.agg_of_node[node]) + i] = 0;
  return out;
}

// extract_block_jacobi(BlockCsrMatrix<float>) (block_jacobi.hpp:72-85) on the
// float-rounded blocks, inverse rounded to float.
std::vector<float> bcsr_block_jacobi_f32(const BcsrD& a) {
  std::vector<float> inv(9 * static_cast<size_t>(a.n));
  for (int32_t r = 0; r < a.n; ++r) {
    double d[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    for (int32_t e = a.row_ptr[r]; e < a.row_ptr[r + 1]; ++e)
      if (a.col_idx[e] == r) {
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) d[i][j] = double(static_cast<float>(a.blocks[9 * size_t(e) + 3 * i + j]));
        break;
      }
    double scale = 0.0, iv[3][3];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) scale = std::max(scale, std::abs(d[i][j]));
    if (scale == 0.0 || !invert3(d, iv, 1e-300))
      validation("block jacobi: singular diagonal block at node " + std::to_string(r));
    for (int q = 0; q < 9; ++q) inv[9 * size_t(r) + q] = static_cast<float>(iv[q / 3][q % 3]);
  }
  return inv;
}

Level2Host build_level2_host(const Mesh& m, const std::vector<double>& lam_e, const std::vector<double>& mu_e,
                             const std::vector<uint8_t>& mask1, int32_t aggregate_target) {
  const BcsrD k1 = assemble_tet4(m, lam_e, mu_e, mask1);
  setup_mark("level2: K1 assembly");
  Aggregation agg = aggregate_p1(k1, aggregate_target);
  setup_mark("level2: aggregation");
  const BcsrD a2 = build_level2(k1, agg, mask1);
  setup_mark("level2: Galerkin");
  Level2Host out;
  out.n2 = agg.n_aggregates;
  out.row_ptr = a2.row_ptr;
  out.col_idx.assign(a2.col_idx.begin(), a2.col_idx.end());
  out.blocks.resize(a2.blocks.size());
  for (size_t q = 0; q < a2.blocks.size(); ++q) out.blocks[q] = static_cast<float>(a2.blocks[q]);
  out.m2 = bcsr_block_jacobi_f32(a2);
  out.mask2 = coarse_mask(agg, mask1);
  out.agg_of_node = std::move(agg.agg_of_node);
  out.seeds = std::move(agg.seeds);
  return out;
}

}  // namespace tsg
