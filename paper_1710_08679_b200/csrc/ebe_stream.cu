// ebe_stream.cu — f = K u from HOST buffers with the PCIe transfers overlapped
// with the sweep (the e2e path behind ts_ebe_apply_host, EbeOperator::apply on
// host VectorBatch data, ebe_operator.hpp:90-134).
//
// Copy-apply-copy moves 3·N·r·s bytes up, sweeps, and moves the same back: at
// 10M DOF × 16 fp32 cases that is 2 × 650 MB over PCIe around a ~1.2 ms sweep,
// so the transfers are the whole cost. The sweep's units (fans or pairs) go in element
// order (slab-major Morton, ebe.cu), so cutting them into chunks gives each node
// a first chunk that reads it and a last chunk that writes it. The schedule then
// runs three streams:
//   in:   u rows whose first reader is chunk k, then event in[k]
//   comp: wait in[k]; constrained identity rows first-read in chunk k; sweep of
//         chunk k (RED into f, zero-filled once up front); event done[k]
//   out:  wait done[k]; f rows whose last writer is chunk k
// so H2D of later rows, the sweep, and D2H of finished rows proceed together
// (PCIe is full duplex). Rows move in contiguous blocks (at most 2 x 1024
// copies); a mesh whose numbering has no locality still gets a correct, if
// less overlapped, schedule.
#include <algorithm>
#include <cstring>

#include "ebe.h"

namespace tsg {
namespace {

constexpr int kMinUnitsPerChunk = 4096;
constexpr int32_t kBlocks = 1024;

template <typename T>
__global__ void k_identity_dofs(const int32_t* __restrict__ dofs, int32_t n, int32_t batch, const T* __restrict__ u,
                                T* __restrict__ f) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= int64_t(n) * batch) return;
  const int64_t at = int64_t(__ldg(dofs + i / batch)) * batch + i % batch;
  f[at] = u[at];
}

bool is_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// The active unit sweep's node rows per unit, in unit order (fans: every element's
// new rows; pairs: the 14 / 5 gathered rows), with each unit's slab key: the
// lowest vertex id of its first element.
struct UnitRows {
  std::vector<int64_t> ptr;   // [U + 1] into rows
  std::vector<int32_t> rows;  // node ids (rows with all three dofs constrained are left out)
  std::vector<int32_t> lo;    // [U] lowest vertex id of the unit's first element
};

UnitRows unit_rows(const ts_ebe& op) {
  UnitRows R;
  if (op.fan) {
    constexpr int kW = 16;  // ebe_fan.cu step record width
    const int32_t U = op.fan->n_units;
    std::vector<int32_t> uf(size_t(U) + 1);
    TS_CUDA(cudaMemcpy(uf.data(), op.fan->ufirst.get(), uf.size() * sizeof(int32_t), cudaMemcpyDeviceToHost));
    std::vector<int32_t> wv(size_t(uf[U]) * kW);
    TS_CUDA(cudaMemcpy(wv.data(), op.fan->words.get(), wv.size() * sizeof(int32_t), cudaMemcpyDeviceToHost));
    R.ptr.assign(1, 0);
    for (int32_t i = 0; i < U; ++i) {
      int32_t lo = INT32_MAX;
      for (int32_t x = uf[i]; x < uf[i + 1]; ++x) {
        const int32_t* w = wv.data() + kW * size_t(x);
        for (int q = 1; q < 15; ++q) {
          const int32_t v = w[q];
          if (v == -1) continue;
          if ((static_cast<uint32_t>(v) >> 28) == 7u) continue;
          R.rows.push_back(v & 0x0FFFFFFF);
        }
        if (x == uf[i])  // p, q, r0, r1 are the first element's vertices
          for (int q : {1, 2, 4, 7})
            if (w[q] != -1) lo = std::min(lo, w[q] & 0x0FFFFFFF);
      }
      R.lo.push_back(lo);
      R.ptr.push_back(static_cast<int64_t>(R.rows.size()));
    }
    return R;
  }
  const int npe = op.npe;
  const int W = npe == 10 ? 16 : 8, NR = npe == 10 ? 14 : 5;
  const int32_t U = op.pair->n_units;
  std::vector<int32_t> pc(size_t(U) * W);
  TS_CUDA(cudaMemcpy(pc.data(), op.pair->conn.get(), pc.size() * sizeof(int32_t), cudaMemcpyDeviceToHost));
  R.ptr.assign(1, 0);
  for (int32_t i = 0; i < U; ++i) {
    const int32_t* w = pc.data() + size_t(i) * W;
    R.lo.push_back(std::min(std::min(w[0], w[1]), std::min(w[2], w[3])) / 3);
    const uint32_t ma = static_cast<uint32_t>(w[NR]), mb = static_cast<uint32_t>(w[NR + 1]);
    for (int r = 0; r < NR; ++r) {
      const uint32_t bits = r < npe ? (ma >> (3 * r)) & 7u : (mb >> (3 * (r - npe))) & 7u;
      if (bits == 7u) continue;  // row neither gathered nor reduced (e.g. a null B's own rows)
      R.rows.push_back(w[r] / 3);
    }
    R.ptr.push_back(static_cast<int64_t>(R.rows.size()));
  }
  return R;
}

std::unique_ptr<EbeStreamPlan> build_stream_plan(const ts_ebe& op) {
  auto P = std::make_unique<EbeStreamPlan>();
  const int32_t U = ebe_unit_count(op), N = op.n_nodes;
  const int32_t min_units = op.fan ? kMinUnitsPerChunk / 3 : kMinUnitsPerChunk;  // a fan is ~3 pairs of work
  if (U < 2 * min_units) return P;  // small: copy-apply-copy is as fast
  const UnitRows R = unit_rows(op);
  // chunks = the element slabs (ebe.cu): units are in element order, slab-major
  const int64_t V = std::max<int32_t>(1, op.n_vertices);
  P->unit_ptr.assign(1, 0);
  int prev = -1;
  for (int32_t i = 0; i < U; ++i) {
    const int sl = ebe_slab_of(R.lo[i], V, op.n_slabs);
    if (sl < prev) return P;  // not slab-ordered (e.g. grouped partition operators)
    if (sl != prev && i > 0 && i - P->unit_ptr.back() >= min_units) P->unit_ptr.push_back(i);
    prev = sl;
  }
  P->unit_ptr.push_back(U);
  const int K = static_cast<int>(P->unit_ptr.size()) - 1;
  if (K < 2) return P;
  P->chunks = K;
  std::vector<int32_t> first(N, K), last(N, -1);
  for (int k = 0; k < K; ++k)
    for (int32_t i = P->unit_ptr[k]; i < P->unit_ptr[k + 1]; ++i)
      for (int64_t q = R.ptr[i]; q < R.ptr[i + 1]; ++q) {
        const int32_t n = R.rows[q];
        first[n] = std::min(first[n], k);
        last[n] = k;  // chunks are visited in order
      }
  for (int32_t n = 0; n < N; ++n)
    if (last[n] < 0) first[n] = last[n] = 0;  // untouched: identity / zero rows, out after chunk 0
  // Node rows move in kBlocks contiguous blocks: a block goes up before the
  // earliest chunk reading any of its rows and comes back after the latest chunk
  // writing any of them (always safe; at slab granularity only boundary blocks
  // wait). Per-node runs would be exact but interleave at every slab boundary
  // (edge nodes are numbered in the mesh's discovery order).
  const int32_t bs = std::max<int32_t>(1, (N + kBlocks - 1) / kBlocks);
  std::vector<int32_t> bfirst, blast;
  for (int32_t a = 0; a < N; a += bs) {
    const int32_t b = std::min(N, a + bs);
    int32_t lo = K, hi = 0;
    for (int32_t n = a; n < b; ++n) {
      lo = std::min(lo, first[n]);
      hi = std::max(hi, last[n]);
    }
    bfirst.push_back(lo);
    blast.push_back(hi);
  }
  auto runs_of = [&](const std::vector<int32_t>& c, std::vector<int32_t>& ptr, std::vector<std::array<int32_t, 2>>& out) {
    std::vector<std::vector<std::array<int32_t, 2>>> per(K);
    const int32_t nb = static_cast<int32_t>(c.size());
    for (int32_t i = 0; i < nb;) {
      int32_t j = i + 1;
      while (j < nb && c[j] == c[i]) ++j;
      per[c[i]].push_back({i * bs, std::min(N, j * bs)});
      i = j;
    }
    ptr.assign(K + 1, 0);
    out.clear();
    for (int k = 0; k < K; ++k) {
      out.insert(out.end(), per[k].begin(), per[k].end());
      ptr[k + 1] = static_cast<int32_t>(out.size());
    }
  };
  runs_of(bfirst, P->in_ptr, P->in_runs);
  runs_of(blast, P->out_ptr, P->out_runs);
  std::vector<int32_t> block_first(N);
  for (int32_t n = 0; n < N; ++n) block_first[n] = bfirst[n / bs];
  // constrained dofs grouped by the chunk that first reads their node
  P->mdof_ptr.assign(K + 1, 0);
  std::vector<int32_t> md;
  if (op.has_mask) {
    std::vector<std::vector<int32_t>> per(K);
    for (size_t d = 0; d < op.host_mask.size(); ++d)
      if (op.host_mask[d]) per[block_first[d / 3]].push_back(static_cast<int32_t>(d));
    for (int k = 0; k < K; ++k) {
      md.insert(md.end(), per[k].begin(), per[k].end());
      P->mdof_ptr[k + 1] = static_cast<int32_t>(md.size());
    }
  }
  P->mdofs.upload(md);
  TS_CUDA(cudaStreamCreateWithFlags(&P->s_in, cudaStreamNonBlocking));
  TS_CUDA(cudaStreamCreateWithFlags(&P->s_comp, cudaStreamNonBlocking));
  TS_CUDA(cudaStreamCreateWithFlags(&P->s_out, cudaStreamNonBlocking));
  TS_CUDA(cudaEventCreateWithFlags(&P->ev_entry, cudaEventDisableTiming));
  P->ev_in.resize(K);
  P->ev_done.resize(K);
  for (int k = 0; k < K; ++k) {
    TS_CUDA(cudaEventCreateWithFlags(&P->ev_in[k], cudaEventDisableTiming));
    TS_CUDA(cudaEventCreateWithFlags(&P->ev_done[k], cudaEventDisableTiming));
  }
  TS_CUDA(cudaDeviceSynchronize());
  P->usable = true;
  return P;
}

template <typename T>
bool apply_streamed(const ts_ebe& op, const EbeStreamPlan& P, const T* uh, T* fh, int32_t batch) {
  const size_t row = 3 * static_cast<size_t>(batch);  // scalars per node
  T* du = reinterpret_cast<T*>(op.stage_u.get());
  T* df = reinterpret_cast<T*>(op.stage_f.get());
  // probe: does the unit sweep cover this batch width? (an empty range launches nothing)
  if (!ebe_unit_apply_range(op, du, df, batch, P.s_comp, 0, 0)) return false;
  // the pipeline's non-blocking streams start after work already queued on the legacy default
  // stream (e.g. a producer of u or a pending reader of f), as the copy-apply-copy path would
  TS_CUDA(cudaEventRecord(P.ev_entry, nullptr));
  TS_CUDA(cudaStreamWaitEvent(P.s_in, P.ev_entry, 0));
  TS_CUDA(cudaStreamWaitEvent(P.s_comp, P.ev_entry, 0));
  TS_CUDA(cudaStreamWaitEvent(P.s_out, P.ev_entry, 0));
  TS_CUDA(cudaMemsetAsync(df, 0, row * op.n_nodes * sizeof(T), P.s_comp));
  for (int k = 0; k < P.chunks; ++k) {
    for (int32_t q = P.in_ptr[k]; q < P.in_ptr[k + 1]; ++q) {
      const auto [a, b] = P.in_runs[q];
      TS_CUDA(cudaMemcpyAsync(du + a * row, uh + a * row, (b - a) * row * sizeof(T), cudaMemcpyHostToDevice, P.s_in));
    }
    TS_CUDA(cudaEventRecord(P.ev_in[k], P.s_in));
    TS_CUDA(cudaStreamWaitEvent(P.s_comp, P.ev_in[k], 0));
    const int32_t m0 = P.mdof_ptr[k], nm = P.mdof_ptr[k + 1] - m0;
    if (nm > 0) {
      const int64_t n = int64_t(nm) * batch;
      k_identity_dofs<T><<<static_cast<unsigned>((n + 255) / 256), 256, 0, P.s_comp>>>(P.mdofs.get() + m0, nm, batch,
                                                                                        du, df);
      TS_CUDA_LAUNCH();
    }
    ebe_unit_apply_range(op, du, df, batch, P.s_comp, P.unit_ptr[k], P.unit_ptr[k + 1]);
    TS_CUDA(cudaEventRecord(P.ev_done[k], P.s_comp));
    TS_CUDA(cudaStreamWaitEvent(P.s_out, P.ev_done[k], 0));
    for (int32_t q = P.out_ptr[k]; q < P.out_ptr[k + 1]; ++q) {
      const auto [a, b] = P.out_runs[q];
      TS_CUDA(cudaMemcpyAsync(fh + a * row, df + a * row, (b - a) * row * sizeof(T), cudaMemcpyDeviceToHost, P.s_out));
    }
  }
  TS_CUDA(cudaStreamSynchronize(P.s_out));
  TS_CUDA(cudaStreamSynchronize(P.s_comp));
  return true;
}

}  // namespace

void ebe_apply_host(const ts_ebe& op, const void* u, void* f, int32_t batch) {
  if (batch < 1) validation("ebe apply: batch must be >= 1");
  const size_t bytes = 3 * static_cast<size_t>(op.n_nodes) * batch * (op.prec / 8);
  std::lock_guard<std::mutex> lock(op.host_mu);
  op.stage_u.ensure(bytes);
  op.stage_f.ensure(bytes);
  if (op.kernel >= 6 && (op.pair || op.fan) && !op.deterministic && is_pinned(u) && is_pinned(f)) {
    if (!op.stream) op.stream = build_stream_plan(op);
    if (op.stream->usable) {
      const bool done =
          op.prec == 32
              ? apply_streamed<float>(op, *op.stream, static_cast<const float*>(u), static_cast<float*>(f), batch)
              : apply_streamed<double>(op, *op.stream, static_cast<const double*>(u), static_cast<double*>(f), batch);
      if (done) return;
    }
  }
  TS_CUDA(cudaMemcpy(op.stage_u.get(), u, bytes, cudaMemcpyHostToDevice));
  ebe_apply(op, op.stage_u.get(), op.stage_f.get(), batch, nullptr);
  TS_CUDA(cudaMemcpy(f, op.stage_f.get(), bytes, cudaMemcpyDeviceToHost));
}

}  // namespace tsg

EbeStreamPlan::~EbeStreamPlan() {
  if (ev_entry) cudaEventDestroy(ev_entry);
  for (cudaEvent_t e : ev_in) cudaEventDestroy(e);
  for (cudaEvent_t e : ev_done) cudaEventDestroy(e);
  for (cudaStream_t s : {s_in, s_comp, s_out})
    if (s) cudaStreamDestroy(s);
}
