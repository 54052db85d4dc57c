// dist.h — mesh partitioning and the per-rank plan of the partitioned solve
// (SURVEY.md §8e). Host-only; no device needed (tested on CPU).
//
// Elements are split into non-overlapping parts; nodes on part interfaces are
// replicated on every part that touches them. Each rank keeps its elements and
// the nodes they touch (local numbering: ascending global id, so local
// vertices come first exactly as in the global mesh, mesh.hpp:26-42, and the
// level-1 vertex vector stays a prefix of the level-0 vector). Replicated
// ("shared") nodes carry identical values on every rank: after each element
// sweep the ranks exchange their partial sums of shared rows and add them in
// ascending rank order, so all copies agree bit for bit. Dot products count a
// node once, on its owner (the lowest rank touching it).
#pragma once
#include <cstdint>
#include <vector>

#include "ts_common.h"

namespace tsg {

// Recursive coordinate bisection of element centroids into `nparts` parts
// (largest-extent axis, split at the count-proportional median).
std::vector<int32_t> partition_rcb(const Mesh& m, int nparts);

// Exchange plan over a prefix of the local nodes.
struct Halo {
  std::vector<int> nbr;                      // neighbour ranks, ascending
  std::vector<std::vector<int32_t>> rows;    // per neighbour: shared local nodes, ascending global id
  std::vector<int32_t> sh_nodes;             // every shared local node (ascending local id)
  std::vector<int32_t> src_ptr;              // [n_shared + 1]
  std::vector<int32_t> src;                  // rank-ordered sources: -1 = own partial, else (k << 24) | row in rows[k]
  int64_t rows_total() const {
    int64_t t = 0;
    for (const auto& r : rows) t += static_cast<int64_t>(r.size());
    return t;
  }
};

struct DistPlan {
  int rank = 0, nranks = 1;
  std::vector<int32_t> elems;        // global ids of this part's elements (ascending)
  std::vector<int32_t> l2g;          // local node -> global node
  int32_t n_local = 0, n_local_vertices = 0;
  std::vector<uint8_t> owned;        // [n_local] 1 = this rank owns the node
  std::vector<uint8_t> elem_boundary;  // [elems] 1 = touches a shared node
  Halo halo0;                        // over all local nodes (level 0 / outer)
  Halo halo1;                        // over local vertices (level 1)
  Mesh local;                        // local mesh (local node ids; bc lists empty)
  std::vector<uint8_t> mask;         // [3 n_local] local dof mask
};

// Plan of `rank` for an element partition `part` ([E] in [0, nranks)).
// `dof_mask` is the global [3N] mask (nullptr = dirichlet_mask of the mesh).
DistPlan build_dist_plan(const Mesh& m, const uint8_t* dof_mask, const int32_t* part, int nranks, int rank);

}  // namespace tsg
