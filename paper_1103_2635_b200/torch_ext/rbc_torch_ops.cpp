// rbc_torch_ops.cpp -- the hot path as registered PyTorch operators (torch.ops.rbc_b200.*),
// a thin layer over the C-ABI (include/rbc_b200.h): CUDA tensors in, CUDA tensors out, on
// the caller's current stream.  No compute here -- every op is one C-ABI call into the
// sm_100a library (librbc_b200.so), so torch.compile graphs, CUDA graphs and autograd-free
// inference code can call the search like any other op.
//
//   bf_search(Tensor queries, Tensor data, int metric, int k) -> (Tensor ids, Tensor dists)
//       brute_force.py:165-186 bf_search
//   pairwise_distances(Tensor a, Tensor b, int metric) -> Tensor
//       metric.py:57-76 pairwise_distances
//   exact_search(int index, Tensor queries, int k) -> (ids, dists, gamma, pruned_radius,
//                                                      pruned_3gamma, candidates)
//       search.py:150-208 exact_query_batch (SearchStats as tensors)
//   one_shot_search(int index, Tensor queries, int k) -> (ids, dists, gamma)
//       search.py:90-141 one_shot_query_batch
// `index` is the opaque rbc_index handle of a built index (DeviceIndex.handle).
// metric: 0 = l2, 1 = l1 (MetricSpec.code).  Errors raise with rbc_last_error().
#include <ATen/cuda/CUDAContext.h>
#include <torch/library.h>
#include <torch/torch.h>

#include <tuple>

#include "rbc_b200.h"

namespace {

void check_rc(int rc, const char *what) {
    TORCH_CHECK(rc == RBC_OK, what, ": ", rbc_last_error(), " (code ", rc, ")");
}

void check_rows(const at::Tensor &t, const char *name) {
    TORCH_CHECK(t.is_cuda(), name, " must be a CUDA tensor");
    TORCH_CHECK(t.scalar_type() == at::kFloat, name, " must be float32");
    TORCH_CHECK(t.dim() == 2, name, " must be 2-D [rows, d]");
    TORCH_CHECK(t.is_contiguous(), name, " must be contiguous");
}

void *stream_of(const at::Tensor &t) {
    return at::cuda::getCurrentCUDAStream(t.device().index()).stream();
}

std::tuple<at::Tensor, at::Tensor> bf_search(const at::Tensor &queries, const at::Tensor &data, int64_t metric,
                                             int64_t k) {
    check_rows(queries, "queries");
    check_rows(data, "data");
    TORCH_CHECK(queries.size(1) == data.size(1), "queries and data must have the same d");
    auto ids = at::empty({queries.size(0), k}, queries.options().dtype(at::kLong));
    auto dists = at::empty({queries.size(0), k}, queries.options());
    check_rc(rbc_bf_search(queries.data_ptr<float>(), queries.size(0), data.data_ptr<float>(), data.size(0),
                           static_cast<int32_t>(data.size(1)), static_cast<int32_t>(metric),
                           static_cast<int32_t>(k), ids.data_ptr<int64_t>(), dists.data_ptr<float>(),
                           stream_of(queries)),
             "bf_search");
    return {ids, dists};
}

at::Tensor pairwise_distances(const at::Tensor &a, const at::Tensor &b, int64_t metric) {
    check_rows(a, "a");
    check_rows(b, "b");
    TORCH_CHECK(a.size(1) == b.size(1), "a and b must have the same d");
    auto out = at::empty({a.size(0), b.size(0)}, a.options());
    check_rc(rbc_pairwise_distances(a.data_ptr<float>(), a.size(0), b.data_ptr<float>(), b.size(0),
                                    static_cast<int32_t>(a.size(1)), static_cast<int32_t>(metric),
                                    out.data_ptr<float>(), stream_of(a)),
             "pairwise_distances");
    return out;
}

std::tuple<at::Tensor, at::Tensor, at::Tensor, at::Tensor, at::Tensor, at::Tensor> exact_search(
    int64_t index, const at::Tensor &queries, int64_t k) {
    check_rows(queries, "queries");
    TORCH_CHECK(index != 0, "null index handle");
    const int64_t nq = queries.size(0);
    auto ids = at::empty({nq, k}, queries.options().dtype(at::kLong));
    auto dists = at::empty({nq, k}, queries.options());
    auto gamma = at::empty({nq}, queries.options());
    auto prr = at::empty({nq}, queries.options().dtype(at::kInt));
    auto p3 = at::empty({nq}, queries.options().dtype(at::kInt));
    auto cand = at::empty({nq}, queries.options().dtype(at::kLong));
    rbc_search_stats stats{gamma.data_ptr<float>(), prr.data_ptr<int32_t>(), p3.data_ptr<int32_t>(),
                           cand.data_ptr<int64_t>()};
    check_rc(rbc_exact_search(reinterpret_cast<const rbc_index *>(index), queries.data_ptr<float>(), nq,
                              static_cast<int32_t>(k), ids.data_ptr<int64_t>(), dists.data_ptr<float>(), stats,
                              stream_of(queries)),
             "exact_search");
    return {ids, dists, gamma, prr, p3, cand};
}

std::tuple<at::Tensor, at::Tensor, at::Tensor> one_shot_search(int64_t index, const at::Tensor &queries, int64_t k) {
    check_rows(queries, "queries");
    TORCH_CHECK(index != 0, "null index handle");
    const int64_t nq = queries.size(0);
    auto ids = at::empty({nq, k}, queries.options().dtype(at::kLong));
    auto dists = at::empty({nq, k}, queries.options());
    auto gamma = at::empty({nq}, queries.options());
    check_rc(rbc_one_shot_search(reinterpret_cast<const rbc_index *>(index), queries.data_ptr<float>(), nq,
                                 static_cast<int32_t>(k), ids.data_ptr<int64_t>(), dists.data_ptr<float>(),
                                 gamma.data_ptr<float>(), stream_of(queries)),
             "one_shot_search");
    return {ids, dists, gamma};
}

}  // namespace

TORCH_LIBRARY(rbc_b200, m) {
    m.def("bf_search(Tensor queries, Tensor data, int metric, int k) -> (Tensor, Tensor)");
    m.def("pairwise_distances(Tensor a, Tensor b, int metric) -> Tensor");
    m.def("exact_search(int index, Tensor queries, int k) -> (Tensor, Tensor, Tensor, Tensor, Tensor, Tensor)");
    m.def("one_shot_search(int index, Tensor queries, int k) -> (Tensor, Tensor, Tensor)");
}

TORCH_LIBRARY_IMPL(rbc_b200, CUDA, m) {
    m.impl("bf_search", &bf_search);
    m.impl("pairwise_distances", &pairwise_distances);
    m.impl("exact_search", &exact_search);
    m.impl("one_shot_search", &one_shot_search);
}
