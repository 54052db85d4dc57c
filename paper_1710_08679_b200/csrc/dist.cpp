// dist.cpp — recursive coordinate bisection and per-rank partition plans.
#include "dist.h"

#include <algorithm>
#include <array>
#include <numeric>
#include <string>

namespace tsg {

std::vector<int32_t> partition_rcb(const Mesh& m, int nparts) {
  const int32_t E = m.n_elems();
  if (nparts < 1 || nparts > 64) validation("partition: nparts must be in [1, 64]");
  if (E < nparts) validation("partition: fewer elements than parts");
  std::vector<std::array<double, 3>> cen(E);
  for (int32_t e = 0; e < E; ++e)
    for (int c = 0; c < 3; ++c) {
      double x = 0.0;
      for (int a = 0; a < 4; ++a) x += m.coords[3 * size_t(m.tets10[10 * size_t(e) + a]) + c];
      cen[e][c] = 0.25 * x;
    }
  std::vector<int32_t> idx(E), part(E, 0);
  std::iota(idx.begin(), idx.end(), 0);
  // (begin, end, first part, number of parts)
  struct Job {
    int32_t b, e;
    int p0, np;
  };
  std::vector<Job> stack{{0, E, 0, nparts}};
  while (!stack.empty()) {
    const Job j = stack.back();
    stack.pop_back();
    if (j.np == 1) {
      for (int32_t i = j.b; i < j.e; ++i) part[idx[i]] = j.p0;
      continue;
    }
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    for (int32_t i = j.b; i < j.e; ++i)
      for (int c = 0; c < 3; ++c) {
        lo[c] = std::min(lo[c], cen[idx[i]][c]);
        hi[c] = std::max(hi[c], cen[idx[i]][c]);
      }
    int ax = 0;
    for (int c = 1; c < 3; ++c)
      if (hi[c] - lo[c] > hi[ax] - lo[ax]) ax = c;
    const int nl = j.np / 2;
    const int32_t cut = j.b + static_cast<int32_t>((int64_t(j.e - j.b) * nl) / j.np);
    // deterministic median: centroid coordinate, then element id
    std::nth_element(idx.begin() + j.b, idx.begin() + cut, idx.begin() + j.e, [&](int32_t x, int32_t y) {
      return cen[x][ax] < cen[y][ax] || (cen[x][ax] == cen[y][ax] && x < y);
    });
    stack.push_back({j.b, cut, j.p0, nl});
    stack.push_back({cut, j.e, j.p0 + nl, j.np - nl});
  }
  return part;
}

namespace {

// Halo over local nodes [0, limit): `ranks[g]` = bitmask of parts touching global node g.
Halo build_halo(const DistPlan& p, const std::vector<uint64_t>& ranks, int32_t limit) {
  Halo h;
  const uint64_t me = uint64_t(1) << p.rank;
  uint64_t nb_mask = 0;
  for (int32_t i = 0; i < limit; ++i) {
    const uint64_t r = ranks[p.l2g[i]];
    if (r != me) nb_mask |= r & ~me;
  }
  std::vector<int> slot(p.nranks, -1);
  for (int q = 0; q < p.nranks; ++q)
    if (nb_mask & (uint64_t(1) << q)) {
      slot[q] = static_cast<int>(h.nbr.size());
      h.nbr.push_back(q);
    }
  h.rows.resize(h.nbr.size());
  // local order is ascending global id, so these lists are ascending in global id
  for (int32_t i = 0; i < limit; ++i) {
    const uint64_t r = ranks[p.l2g[i]] & ~me;
    if (!r) continue;
    for (int q = 0; q < p.nranks; ++q)
      if (r & (uint64_t(1) << q)) h.rows[slot[q]].push_back(i);
  }
  std::vector<std::vector<int32_t>::const_iterator> cur;
  for (const auto& rw : h.rows) cur.push_back(rw.begin());
  h.src_ptr.push_back(0);
  for (int32_t i = 0; i < limit; ++i) {
    const uint64_t r = ranks[p.l2g[i]];
    if (r == me) continue;
    h.sh_nodes.push_back(i);
    for (int q = 0; q < p.nranks; ++q) {  // ascending rank order
      if (!(r & (uint64_t(1) << q))) continue;
      if (q == p.rank) {
        h.src.push_back(-1);
      } else {
        const int k = slot[q];
        const int32_t pos = static_cast<int32_t>(cur[k] - h.rows[k].begin());
        if (cur[k] == h.rows[k].end() || *cur[k] != i) validation("dist plan: inconsistent halo rows");
        ++cur[k];
        if (k >= 128 || pos >= (1 << 24)) validation("dist plan: halo too large for the source encoding");
        h.src.push_back((k << 24) | pos);
      }
    }
    h.src_ptr.push_back(static_cast<int32_t>(h.src.size()));
  }
  return h;
}

}  // namespace

DistPlan build_dist_plan(const Mesh& m, const uint8_t* dof_mask, const int32_t* part, int nranks, int rank) {
  if (nranks < 1 || nranks > 64) validation("dist plan: nranks must be in [1, 64]");
  if (rank < 0 || rank >= nranks) validation("dist plan: rank out of range");
  const int32_t E = m.n_elems(), N = m.n_nodes(), V = m.vertex_count;
  DistPlan p;
  p.rank = rank;
  p.nranks = nranks;
  std::vector<uint64_t> ranks(N, 0);
  for (int32_t e = 0; e < E; ++e) {
    const int32_t q = part[e];
    if (q < 0 || q >= nranks) validation("dist plan: element " + std::to_string(e) + " has part out of range");
    for (int a = 0; a < 10; ++a) ranks[m.tets10[10 * size_t(e) + a]] |= uint64_t(1) << q;
    if (q == rank) p.elems.push_back(e);
  }
  // local nodes: ascending global id (vertices, which are numbered first globally, stay first)
  std::vector<int32_t> g2l(N, -1);
  for (int32_t e : p.elems)
    for (int a = 0; a < 10; ++a) g2l[m.tets10[10 * size_t(e) + a]] = 1;
  for (int32_t g = 0; g < N; ++g)
    if (g2l[g] == 1) {
      g2l[g] = static_cast<int32_t>(p.l2g.size());
      p.l2g.push_back(g);
      if (g < V) ++p.n_local_vertices;
    }
  p.n_local = static_cast<int32_t>(p.l2g.size());
  p.owned.resize(p.n_local);
  for (int32_t i = 0; i < p.n_local; ++i) {
    const uint64_t r = ranks[p.l2g[i]];
    p.owned[i] = (r & ((uint64_t(1) << rank) - 1)) == 0 ? 1 : 0;  // no lower rank touches it
  }
  p.elem_boundary.resize(p.elems.size());
  const uint64_t me = uint64_t(1) << rank;
  for (size_t k = 0; k < p.elems.size(); ++k) {
    uint8_t b = 0;
    for (int a = 0; a < 10; ++a) b |= ranks[m.tets10[10 * size_t(p.elems[k]) + a]] != me;
    p.elem_boundary[k] = b;
  }
  // local mesh
  Mesh& L = p.local;
  L.vertex_count = p.n_local_vertices;
  L.coords.resize(3 * size_t(p.n_local));
  for (int32_t i = 0; i < p.n_local; ++i)
    for (int c = 0; c < 3; ++c) L.coords[3 * size_t(i) + c] = m.coords[3 * size_t(p.l2g[i]) + c];
  L.tets10.resize(10 * p.elems.size());
  L.material_id.resize(p.elems.size());
  for (size_t k = 0; k < p.elems.size(); ++k) {
    for (int a = 0; a < 10; ++a) L.tets10[10 * k + a] = g2l[m.tets10[10 * size_t(p.elems[k]) + a]];
    L.material_id[k] = m.material_id[p.elems[k]];
  }
  const std::vector<uint8_t> gm = dof_mask ? std::vector<uint8_t>() : m.dirichlet_mask();
  const uint8_t* mk = dof_mask ? dof_mask : gm.data();
  p.mask.resize(3 * size_t(p.n_local));
  for (int32_t i = 0; i < p.n_local; ++i)
    for (int c = 0; c < 3; ++c) p.mask[3 * size_t(i) + c] = mk[3 * size_t(p.l2g[i]) + c];
  p.halo0 = build_halo(p, ranks, p.n_local);
  p.halo1 = build_halo(p, ranks, p.n_local_vertices);
  return p;
}

}  // namespace tsg
