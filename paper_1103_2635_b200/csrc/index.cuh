// index.cuh -- the device-resident RBC index behind the opaque rbc_index.
#pragma once

#include "common.cuh"

struct rbc_index {
    int kind = 0;  // 0 = exact (RbcExactIndex), 1 = one-shot (RbcOneShotIndex)
    int64_t n = 0;
    int d = 0;
    int metric = 0;
    int64_t nr = 0;
    int s = 0;
    bool shard = false;
    int device = 0;
    size_t bytes = 0;

    float *x = nullptr;        // [n, d] database, point-id order
    float *reps = nullptr;     // [nr, d] representative rows X[rep_ids]
    int64_t *rep_ids = nullptr;
    float *radii = nullptr;    // [nr] list radii psi_r

    // exact: lists in CSR (representative-position order), list-ordered copy
    int64_t *offsets = nullptr;  // [nr + 1]
    int32_t *perm = nullptr;     // [n_local] point id of each list entry
    float *list_dists = nullptr; // [n_local] dist to the owning rep (ascending per list)
    float *xp = nullptr;         // [n_local, d] X[perm]
    int64_t n_local = 0;         // entries held (== n unless a shard)

    // tensor-core stage-2 operands (tc_scan.cu): per list, rows centred on
    // the list's rep, fp16, pre-swizzled for the UMMA shared-memory layout
    void *tc = nullptr;
    // tensor-core stage-1 operands (tc_stage1.cu): representatives centred on
    // their mean, f16, pre-swizzled
    void *tc1 = nullptr;

    // one-shot: [nr, s] point ids
    int32_t *lists = nullptr;

    // fp32 SIMT filter operands (simt_scan.cu), rows padded to d4 = d rounded up to 4:
    // the representatives and (one-shot) the s-lists' rows gathered per list
    float *reps4 = nullptr;  // [nr, d4]
    float *x4 = nullptr;     // [nr * s, d4]

    // stage-2 work-item capacity learned from previous searches (tile unions)
    mutable int64_t s2_work_per_tile = 24;

    // captured fused-search graph + its scratch arena (search.cu), reused while a
    // caller repeats the same (queries, nq, k, outputs) call
    mutable void *graph = nullptr;
    // device buffers of the host-buffer search entry points (abi.cu), grown on demand
    mutable void *hostbuf = nullptr;
};

namespace rbc {
int tc_index_prepare(rbc_index *idx, cudaStream_t st);
void tc_index_release(rbc_index *idx);
int tc1_index_prepare(rbc_index *idx, cudaStream_t st);
void tc1_index_release(rbc_index *idx);
void search_graph_release(const rbc_index *idx);
void host_buffers_release(const rbc_index *idx);
}  // namespace rbc
