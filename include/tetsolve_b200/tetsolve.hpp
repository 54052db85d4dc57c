// tetsolve_b200/tetsolve.hpp — umbrella over the drop-in headers
// include/tetsolve/<module>.hpp, which keep the reference's module names
// (/root/reference/proj/include/tetsolve): a reference user keeps its
// `#include "tetsolve/adaptive_cg.hpp"` etc., points -I at this repo's
// include/ and links libtsgpu.so (include/tsgpu.h). Types, signatures,
// ownership (value types, host VectorBatch in/out) and exceptions follow the
// reference; all arithmetic runs on the GPU.
#pragma once

#include "../tetsolve/errors.hpp"
#include "../tetsolve/geometry.hpp"
#include "../tetsolve/material.hpp"
#include "../tetsolve/mesh.hpp"
#include "../tetsolve/box_mesh.hpp"
#include "../tetsolve/vector_batch.hpp"
#include "../tetsolve/block_csr.hpp"
#include "../tetsolve/block_jacobi.hpp"
#include "../tetsolve/prolongation.hpp"
#include "../tetsolve/ebe_operator.hpp"
#include "../tetsolve/pcg.hpp"
#include "../tetsolve/solver_config.hpp"
#include "../tetsolve/aggregation.hpp"
#include "../tetsolve/adaptive_cg.hpp"
#include "../tetsolve/fault.hpp"
#include "../tetsolve/model.hpp"
#include "../tetsolve/greens.hpp"
#include "../tetsolve/mesh_io.hpp"
#include "../tetsolve/solution_io.hpp"
