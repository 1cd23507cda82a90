// B200 mirror of the reference loss-side API (/root/reference/proj/include/seqpar/losses.hpp,
// exact_sum.hpp, the reduction half of comm.hpp): per-position log-probs on the GPU, exact
// order-independent sums, and the group reductions the sharded losses are built from. The
// autograd wiring (grad-aware vs plain backward, SFT / DPO losses) is in the Python package
// (paper_2505_22296_b200/losses.py) on top of these entry points.
#pragma once
#include <cuda_runtime.h>

#include <array>
#include <cstdint>
#include <vector>

#include "seqpar/comm.hpp"
#include "seqpar/partition.hpp"

namespace seqpar {

// exact_sum.hpp: 2240-bit two's-complement fixed point in units of 2^-1074 — exact for any
// finite doubles, so sums are independent of order and sharding; rounds once (RNE).
class ExactSum {
 public:
  static constexpr int kLimbs = 35;
  void add(double v);
  void merge(const ExactSum& other);
  double round_to_double() const;
  bool is_zero() const;
  const std::array<uint64_t, kLimbs>& limbs() const { return limbs_; }
  static ExactSum from_limbs(const std::array<uint64_t, kLimbs>& limbs);

 private:
  std::array<uint64_t, kLimbs> limbs_{};
};

// Exact sum of n device doubles (one-block kernel, per-thread accumulators merged pairwise).
ExactSum exact_sum_device(const double* values, int64_t n, cudaStream_t s);

// sequence_logprob_per_position (losses.cpp:20-72) on device: logits [T, V] of dtype
// 0 fp32 / 1 bf16 / 2 fp64,
// labels [T] int64 (kIgnoreLabel -> 0 and no gradient); out / lse [T] fp64. The backward
// writes (or adds into) dlogits = g_t * (onehot(label) - softmax(row)).
void logprob_forward(cudaStream_t s, const void* logits, int dtype, int64_t T, int64_t V,
                     const int64_t* labels, double* out, double* lse);
void logprob_backward(cudaStream_t s, const void* logits, int dtype, int64_t T, int64_t V,
                      const int64_t* labels, const double* lse, const double* g, void* dlogits,
                      bool accumulate);

// Group reductions over the rank's transport (comm.cpp:339-353, :504-524), counted like the
// reference: exact accumulators, int64 counts, small f64 vectors (balanced tree sum in group
// order, tree_sum_into comm.cpp:323-337).
ExactSum exact_sum_all_reduce(RankCtx& ctx, const CommGroup& group, const ExactSum& local);
int64_t all_reduce_count(RankCtx& ctx, const CommGroup& group, int64_t n);
std::vector<double> all_reduce_values(RankCtx& ctx, const CommGroup& group, const std::vector<double>& vals);
// all-gather of equal-size host payloads (device staging over the transport)
std::vector<std::vector<uint8_t>> exchange_host(RankCtx& ctx, const CommGroup& group, const void* data,
                                                size_t bytes);

}  // namespace seqpar
