// tc_scan.cuh -- dispatch of the distance scans: the tcgen05 stage-1/stage-2
// engines (tensor-core filter + exact fp64 re-rank, tc_stage1.cu / tc_stage2.cu)
// and the exact fp64 SIMT scans (exact_kernels.cu) they fall back to.
#pragma once

#include "common.cuh"
#include "index.cuh"

namespace rbc {

struct PruneOut;

// k=1 key64 argmin of every q row over the rows of x (build assignment,
// one-shot nearest rep, bf_search k=1).  keys[i] = (f32 bits(dist) << 32) | j.
// x4: optional copy of x with rows padded to d rounded up to 4 (the SIMT engine's layout)
int nearest_rows(const float *q, int64_t nq, const float *x, int64_t n, int d, int metric, uint64_t *keys,
                 cudaStream_t st, const float *x4 = nullptr);

// bf_search core: k nearest keys per query row over all of x, sorted.
int bf_search_keys(const float *q, int64_t nq, const float *x, int64_t n, int d, int metric, int k, uint64_t *keys,
                   cudaStream_t st);

// Range guard of the tensor-core engines: their fp32 bounds (squared norms, the error terms)
// stay finite only while every coordinate is at most kTcMaxAbs in magnitude (d <= 128:
// 512 kTcMaxAbs^2 << FLT_MAX).  Index operands are checked when they are prepared, queries per
// call (synchronising: one max-reduce); out-of-range data takes the SIMT / exact engines,
// which accumulate in fp64 or treat an overflowed fp32 bound as undecided.
constexpr float kTcMaxAbs = 1e15f;
bool tc_range_ok(const float *a, int64_t count, cudaStream_t st);

// stage 1 of the searches: bit-exact dist(q_i, r_p) -> d1[nq, nr]
int stage1_distances(const rbc_index *idx, const float *q, int64_t nq, float *d1, cudaStream_t st);

// filtered stage 1 + pruning (filter_stage1.cu) for indexes without the tensor-core stage 1
// (d > 64, L1): fp32 SIMT bounds for every (q, r), exact fp64 only where a decision needs it.
// d1 [nq, nr] and len [nq, nr] are scratch; ok = false (a query with too many gamma
// candidates): nothing usable was produced and the caller runs stage1_distances + prune.
bool filter_stage1_supported(const rbc_index *idx, int k);
int64_t filter_stage1_stride(int64_t nr);  // row stride of d1 / len (16-byte rows)
int filter_stage1(const rbc_index *idx, const float *q, int64_t nq, int k, float *d1, int32_t *len, PruneOut &out,
                  bool &ok, cudaStream_t st);

// stage 2 of the exact search over the pruned segments (synchronising wrapper
// around tc_stage2 / stage2_exact)
int stage2_scan(const rbc_index *idx, const float *q, int64_t nq, int k, const PruneOut &po, uint64_t *keys,
                cudaStream_t st);

// tcgen05 stage 1 + pruning (tc_stage1.cu), stream-ordered, no host sync;
// *fail_dev (device int) becomes nonzero when a buffer overflowed and the
// caller must redo the batch with the exact path
bool tc_stage1_supported(const rbc_index *idx, int k);
int tc_stage1(const rbc_index *idx, const float *q, int64_t nq, int k, PruneOut &out, int32_t *fail_dev,
              cudaStream_t st);
// rows of src [rows][d] -> dst [rows][64], zero padded
void pad_rows64(const float *src, int64_t rows, int d, float *dst, cudaStream_t st);

// tcgen05 stage 2 (tc_stage2.cu)
bool tc_stage2_supported(const rbc_index *idx, int k);
// stream-ordered, no host sync: work arrays sized cap_work; writes
// status_dev[0] = work items needed (> cap_work: results invalid, re-run),
// status_dev[1] = queries recomputed by the exact overflow scan
int tc_stage2(const rbc_index *idx, const float *q, int64_t nq, int k, const PruneOut &po, uint64_t *keys,
              int64_t cap_work, int64_t *status_dev, cudaStream_t st, int cap_groups = 0);

// tcgen05 brute force (tc_stage2.cu): k nearest keys of every q row over all rows of x,
// sorted, bit-identical to the exact scan (L2, d <= 64, k <= 16)
bool tc_bf_supported(int64_t nq, int64_t n, int d, int metric, int k);
int tc_bf_keys(const float *q, int64_t nq, const float *x, int64_t n, int d, int k, uint64_t *keys, cudaStream_t st);
// tcgen05 brute force over a prepared (partitioned, kind 2) operand: every list, every query
int tc_bf_index_search(const rbc_index *idx, const float *q, int64_t nq, int k, uint64_t *keys, cudaStream_t st);
// tcgen05 one-shot list scan (tc_stage2.cu): operands of the s-lists (xp_lists = the
// points of every list, gathered, [nr * s][d]) and the scan of each query's own list
int tc_one_shot_prepare(rbc_index *idx, const float *xp_lists, cudaStream_t st);
bool tc_one_shot_supported(const rbc_index *idx, int64_t nq, int k);
int tc_one_shot_scan(const rbc_index *idx, const float *q, int64_t nq, int k, const uint64_t *near, uint64_t *keys,
                     cudaStream_t st);
// prepared brute-force operand (abi.cu) and when preparing one per call pays off
int bf_prepare(const float *x, int64_t n, int d, int metric, rbc_index **out, cudaStream_t st);
bool bf_partition_pays(int64_t nq, int64_t n, int d, int metric, int k);
int64_t &last_overflow_count();
// stage-2 work-item capacity for nq queries, and its update from a measured need
int64_t stage2_work_capacity(const rbc_index *idx, int64_t nq);
void stage2_note_work(const rbc_index *idx, int64_t nq, int64_t needed);

// fp32 SIMT filter + exact fp64 re-rank (simt_scan.cu): the L1 engine, and L2 where the
// tensor-core scans do not apply (d <= 128, k <= 32)
bool simt_supported(int d, int k);
bool simt_one_shot_supported(const rbc_index *idx, int64_t nq, int k);
int simt_dense_topk(const float *q, int64_t nq, const float *x, int64_t n, int d, int metric, int k,
                    const int32_t *pid, uint64_t *keys, cudaStream_t st, const float *x4 = nullptr);
int simt_index_prepare(rbc_index *idx, cudaStream_t st);
// exact-search stage 2 on the SIMT filter (L1 exact indexes): the surviving segments (CSR per
// query: seg_off, nseg; per segment its list and cutoff; `total` segments) -> k keys per query
bool simt_exact_supported(const rbc_index *idx, int64_t nq, int k);
int simt_exact_stage2(const rbc_index *idx, const float *q, int64_t nq, int k, const int64_t *seg_off,
                      const int32_t *nseg, const int32_t *seg_list, const int32_t *seg_len, const float *gamma,
                      int64_t total, uint64_t *keys, cudaStream_t st);
int simt_one_shot_scan(const rbc_index *idx, const float *q, int64_t nq, int k, const uint64_t *near, uint64_t *keys,
                       cudaStream_t st);

// k nearest keys for large k (select.cu): a sampled fp32 threshold, one counting and
// collecting pass, a segmented sort of the collected exact keys (k > 32)
bool select_large_supported(int64_t nq, int64_t n, int d, int k);
int select_topk_large(const float *q, int64_t nq, const float *x, int64_t n, int d, int metric, int k, uint64_t *keys,
                      cudaStream_t st);

// engine selection (RBC_ENGINE env: "auto" (default) | "exact")
bool force_exact_engine();
// minimum (query, point) pairs for the brute-force-shaped tensor-core scans (0 in mode 2)
int64_t tc_min_pairs();
// minimum (query, point) pairs for the fp32 SIMT filter scans (0 in modes 2 and 3)
int64_t simt_min_pairs();

}  // namespace rbc
