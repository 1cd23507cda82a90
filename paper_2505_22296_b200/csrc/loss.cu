// The step after the model: per-position label log-probabilities and the sharded loss
// reductions of the SP group (reference proj/src/losses.cpp, exact_sum.cpp, comm.cpp:464-524).
//
//   * logprob_fwd / logprob_bwd kernels: one CTA per sequence position, online max/sum of the
//     row in fp64 (the reference computes in f64, losses.cpp:20-50), fp32 or bf16 logits; the
//     backward writes g * (onehot(label) - softmax) (losses.cpp:52-70). HBM-bound row streams.
//   * ExactSum: a 2240-bit two's-complement fixed-point accumulator in units of 2^-1074
//     (exact_sum.hpp), so a sum is independent of order and of the sharding. The device kernel
//     gives every thread its own accumulator in shared memory, then merges them pairwise.
//   * group reductions over the transport (NCCL or loopback): all-gather of the 280-byte
//     accumulators / int64 counts / small f64 vectors, combined on the host in group order
//     (tree order for f64 values, comm.cpp:323-353), counted as the reference counts them.
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "seqpar/losses.hpp"

namespace seqpar {

#define LS_CUDA(x)                                                                            \
  do {                                                                                        \
    cudaError_t e_ = (x);                                                                     \
    if (e_ != cudaSuccess) throw StateError(std::string("CUDA: ") + cudaGetErrorString(e_) + \
                                            " at " #x);                                       \
  } while (0)

// ------------------------------------------------------------------------------ ExactSum
namespace {

__host__ __device__ inline void limb_add(uint64_t* x, int limb, uint64_t chunk) {
  for (int i = limb; chunk && i < ExactSum::kLimbs; ++i) {
    const uint64_t before = x[i];
    x[i] = before + chunk;
    chunk = x[i] < before ? 1 : 0;
  }
}
__host__ __device__ inline void limb_sub(uint64_t* x, int limb, uint64_t chunk) {
  for (int i = limb; chunk && i < ExactSum::kLimbs; ++i) {
    const uint64_t before = x[i];
    x[i] = before - chunk;
    chunk = before < chunk ? 1 : 0;
  }
}
// |v| = m * 2^(e - 1074) with m < 2^53 an integer: two 64-bit chunks at limb offset e / 64
__host__ __device__ inline void exact_add(uint64_t* x, double v) {
  if (v == 0.0) return;
  uint64_t bits;
  memcpy(&bits, &v, sizeof(bits));
  const int bexp = static_cast<int>((bits >> 52) & 0x7ff);
  uint64_t m = bits & ((1ull << 52) - 1);
  int e;  // bit offset of m's LSB in units of 2^-1074
  if (bexp == 0) {
    e = 0;  // subnormal: m * 2^-1074
  } else {
    m |= 1ull << 52;
    e = bexp - 1;
  }
  const int limb = e / 64, off = e % 64;
  const uint64_t lo = m << off, hi = off ? (m >> (64 - off)) : 0;
  if (bits >> 63) {
    limb_sub(x, limb, lo);
    limb_sub(x, limb + 1, hi);
  } else {
    limb_add(x, limb, lo);
    limb_add(x, limb + 1, hi);
  }
}
__host__ __device__ inline void exact_merge(uint64_t* x, const uint64_t* y) {
  uint64_t carry = 0;
  for (int i = 0; i < ExactSum::kLimbs; ++i) {
    const uint64_t a = x[i], s = a + y[i];
    const uint64_t c1 = s < a ? 1 : 0;
    x[i] = s + carry;
    carry = c1 | (x[i] < s ? 1 : 0);
  }
}

// One block: thread t accumulates values t, t + blockDim, ... into its own accumulator in
// shared memory; accumulators merge pairwise (exact, so the tree order does not matter).
// out[kLimbs] = 1 when any value is Inf / NaN (exponent field 0x7ff): the host then throws like
// ExactSum::add (exact_sum.cpp) instead of returning a sum of garbage fixed-point chunks.
__global__ void exact_sum_kernel(const double* v, int64_t n, uint64_t* out) {
  extern __shared__ uint64_t acc[];  // [blockDim][kLimbs]
  uint64_t* mine = acc + threadIdx.x * ExactSum::kLimbs;
  for (int i = 0; i < ExactSum::kLimbs; ++i) mine[i] = 0;
  int bad = 0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double x = v[i];
    if (((__double_as_longlong(x) >> 52) & 0x7ff) == 0x7ff) {
      bad = 1;
      continue;
    }
    exact_add(mine, x);
  }
  bad = __syncthreads_or(bad);
  if (threadIdx.x == 0) out[ExactSum::kLimbs] = bad;
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) exact_merge(mine, acc + (threadIdx.x + s) * ExactSum::kLimbs);
    __syncthreads();
  }
  if (threadIdx.x < ExactSum::kLimbs) out[threadIdx.x] = acc[threadIdx.x];
}

// ---------------------------------------------------------------------------- log-probs
template <typename T>
__device__ __forceinline__ double ld(const T* p, int64_t i);
template <>
__device__ __forceinline__ double ld<float>(const float* p, int64_t i) { return p[i]; }
template <>
__device__ __forceinline__ double ld<double>(const double* p, int64_t i) { return p[i]; }
template <>
__device__ __forceinline__ double ld<__nv_bfloat16>(const __nv_bfloat16* p, int64_t i) {
  return __bfloat162float(p[i]);
}

// (max, sum of exp(x - max)) pairs merge like the attention online softmax
__device__ __forceinline__ void lse_merge(double& m, double& s, double m2, double s2) {
  if (m2 == -INFINITY) return;
  if (m == -INFINITY) {
    m = m2, s = s2;
    return;
  }
  const double mx = fmax(m, m2);
  s = s * exp(m - mx) + s2 * exp(m2 - mx);
  m = mx;
}

template <typename T>
__global__ void __launch_bounds__(256) logprob_fwd_kernel(const T* logits, int64_t V, const int64_t* labels,
                                                          double* out, double* lse_out) {
  const int64_t t = blockIdx.x;
  const int64_t lab = labels[t];
  if (lab == kIgnoreLabel) {  // unsupervised: 0, no gradient (losses.cpp:34)
    if (threadIdx.x == 0) out[t] = 0.0, lse_out[t] = 0.0;
    return;
  }
  const T* row = logits + t * V;
  double m = -INFINITY, s = 0.0;
  for (int64_t j = threadIdx.x; j < V; j += blockDim.x) {
    const double x = ld(row, j);
    if (x > m) {
      s = (m == -INFINITY ? 0.0 : s * exp(m - x)) + 1.0;
      m = x;
    } else {
      s += exp(x - m);
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, s, o);
    lse_merge(m, s, m2, s2);
  }
  __shared__ double sm[8], ss[8];
  const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (lane == 0) sm[w] = m, ss[w] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < (int)blockDim.x / 32; ++i) lse_merge(m, s, sm[i], ss[i]);
    const double lse = m + log(s);
    lse_out[t] = lse;
    out[t] = ld(row, lab) - lse;
  }
}

template <typename T>
__global__ void __launch_bounds__(256) logprob_bwd_kernel(const T* logits, int64_t V, const int64_t* labels,
                                                          const double* lse, const double* g, T* dlogits,
                                                          int accumulate) {
  const int64_t t = blockIdx.x;
  const int64_t lab = labels[t];
  const double gt = lab == kIgnoreLabel ? 0.0 : g[t];
  const T* row = logits + t * V;
  T* drow = dlogits + t * V;
  for (int64_t j = threadIdx.x; j < V; j += blockDim.x) {
    double d = gt == 0.0 ? 0.0 : -gt * exp(ld(row, j) - lse[t]);
    if (j == lab) d += gt;
    if (accumulate) d += ld(drow, j);
    if constexpr (sizeof(T) == 8)
      drow[j] = d;
    else if constexpr (sizeof(T) == 4)
      drow[j] = static_cast<float>(d);
    else
      drow[j] = __double2bfloat16(d);
  }
}

}  // namespace

void ExactSum::add(double v) {
  if (!std::isfinite(v)) throw ConfigError("ExactSum requires finite values");
  exact_add(limbs_.data(), v);
}
void ExactSum::merge(const ExactSum& o) { exact_merge(limbs_.data(), o.limbs_.data()); }
bool ExactSum::is_zero() const {
  for (uint64_t l : limbs_)
    if (l) return false;
  return true;
}
ExactSum ExactSum::from_limbs(const std::array<uint64_t, kLimbs>& limbs) {
  ExactSum s;
  s.limbs_ = limbs;
  return s;
}

// Round-to-nearest-even of the exact fixed-point value (exact_sum.hpp's round_to_double).
double ExactSum::round_to_double() const {
  std::array<uint64_t, kLimbs> mag = limbs_;
  const bool neg = mag[kLimbs - 1] >> 63;
  if (neg) {  // two's complement magnitude
    for (auto& l : mag) l = ~l;
    limb_add(mag.data(), 0, 1);
  }
  int top = -1;
  for (int i = kLimbs - 1; i >= 0 && top < 0; --i)
    if (mag[static_cast<size_t>(i)]) top = i * 64 + 63 - __builtin_clzll(mag[static_cast<size_t>(i)]);
  if (top < 0) return 0.0;
  auto bit = [&](int p) -> uint64_t { return p < 0 ? 0 : (mag[static_cast<size_t>(p / 64)] >> (p % 64)) & 1; };
  // 53 significant bits starting at `top` (fewer when the value is subnormal-sized)
  const int lsb = top - 52 > 0 ? top - 52 : 0;
  uint64_t mant = 0;
  for (int p = top; p >= lsb; --p) mant = (mant << 1) | bit(p);
  int e = lsb;  // value = mant * 2^(e - 1074) (+ rounding)
  if (lsb > 0) {
    const uint64_t half = bit(lsb - 1);
    bool rest = false;
    for (int p = lsb - 2; p >= 0 && !rest; --p) rest = bit(p) != 0;
    if (half && (rest || (mant & 1))) {
      if (++mant == (1ull << 53)) mant >>= 1, ++e;
    }
  }
  const double v = std::ldexp(static_cast<double>(mant), e - 1074);
  return neg ? -v : v;
}

ExactSum exact_sum_device(const double* values, int64_t n, cudaStream_t s) {
  ExactSum r;
  if (n <= 0) return r;
  uint64_t* d = nullptr;
  LS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d), (ExactSum::kLimbs + 1) * 8, s));
  constexpr int kThreads = 128;
  exact_sum_kernel<<<1, kThreads, kThreads * ExactSum::kLimbs * 8, s>>>(values, n, d);
  spattn::note_launch();
  LS_CUDA(cudaGetLastError());
  std::array<uint64_t, ExactSum::kLimbs + 1> h{};
  LS_CUDA(cudaMemcpyAsync(h.data(), d, sizeof(h), cudaMemcpyDeviceToHost, s));
  LS_CUDA(cudaFreeAsync(d, s));
  LS_CUDA(cudaStreamSynchronize(s));
  if (h[ExactSum::kLimbs]) throw ConfigError("ExactSum requires finite values");
  std::array<uint64_t, ExactSum::kLimbs> limbs{};
  for (int i = 0; i < ExactSum::kLimbs; ++i) limbs[static_cast<size_t>(i)] = h[static_cast<size_t>(i)];
  return ExactSum::from_limbs(limbs);
}

void logprob_forward(cudaStream_t s, const void* logits, int dtype, int64_t T, int64_t V,
                     const int64_t* labels, double* out, double* lse) {
  if (T == 0) return;
  if (V <= 0) throw ShapeError("sequence_logprob: empty vocabulary");
  switch (dtype) {
    case 0: logprob_fwd_kernel<float><<<(unsigned)T, 256, 0, s>>>(static_cast<const float*>(logits), V, labels, out, lse); break;
    case 1: logprob_fwd_kernel<__nv_bfloat16><<<(unsigned)T, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(logits), V, labels, out, lse); break;
    case 2: logprob_fwd_kernel<double><<<(unsigned)T, 256, 0, s>>>(static_cast<const double*>(logits), V, labels, out, lse); break;
    default: throw ConfigError("sequence_logprob: dtype must be 0 (fp32), 1 (bf16) or 2 (fp64)");
  }
  spattn::note_launch();
  LS_CUDA(cudaGetLastError());
}

void logprob_backward(cudaStream_t s, const void* logits, int dtype, int64_t T, int64_t V,
                      const int64_t* labels, const double* lse, const double* g, void* dlogits,
                      bool accumulate) {
  if (T == 0) return;
  const int acc = accumulate ? 1 : 0;
  switch (dtype) {
    case 0: logprob_bwd_kernel<float><<<(unsigned)T, 256, 0, s>>>(static_cast<const float*>(logits), V, labels, lse, g, static_cast<float*>(dlogits), acc); break;
    case 1: logprob_bwd_kernel<__nv_bfloat16><<<(unsigned)T, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(logits), V, labels, lse, g, static_cast<__nv_bfloat16*>(dlogits), acc); break;
    case 2: logprob_bwd_kernel<double><<<(unsigned)T, 256, 0, s>>>(static_cast<const double*>(logits), V, labels, lse, g, static_cast<double*>(dlogits), acc); break;
    default: throw ConfigError("sequence_logprob: dtype must be 0 (fp32), 1 (bf16) or 2 (fp64)");
  }
  spattn::note_launch();
  LS_CUDA(cudaGetLastError());
}

// --------------------------------------------------------------------- group reductions
// All-gather of equal-size host payloads over the transport (device staging).
std::vector<std::vector<uint8_t>> exchange_host(RankCtx& ctx, const CommGroup& group, const void* data,
                                                size_t bytes) {
  const int g = group.size(), me = group.index_of(ctx.rank);
  std::vector<std::vector<uint8_t>> out(static_cast<size_t>(g));
  out[static_cast<size_t>(me)].assign(static_cast<const uint8_t*>(data), static_cast<const uint8_t*>(data) + bytes);
  if (g == 1 || bytes == 0) {
    for (auto& o : out) o.resize(bytes);
    return out;
  }
  cudaStream_t s = ctx.stream;
  uint8_t* buf = nullptr;
  LS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&buf), bytes * static_cast<size_t>(g), s));
  uint8_t* mine = buf + bytes * static_cast<size_t>(me);
  LS_CUDA(cudaMemcpyAsync(mine, data, bytes, cudaMemcpyHostToDevice, s));
  std::vector<Msg> sends, recvs;
  for (int j = 0; j < g; ++j) {
    if (j == me) continue;
    sends.push_back({j, mine, bytes});
    recvs.push_back({j, buf + bytes * static_cast<size_t>(j), bytes});
  }
  ctx.transport->send_recv(group, ctx.rank, sends, recvs, s);
  std::vector<uint8_t> all(bytes * static_cast<size_t>(g));
  LS_CUDA(cudaMemcpyAsync(all.data(), buf, all.size(), cudaMemcpyDeviceToHost, s));
  LS_CUDA(cudaFreeAsync(buf, s));
  LS_CUDA(cudaStreamSynchronize(s));
  for (int j = 0; j < g; ++j)
    out[static_cast<size_t>(j)].assign(all.begin() + static_cast<int64_t>(bytes) * j,
                                       all.begin() + static_cast<int64_t>(bytes) * (j + 1));
  return out;
}

ExactSum exact_sum_all_reduce(RankCtx& ctx, const CommGroup& group, const ExactSum& local) {
  const int g = group.size();
  ctx.count(Primitive::all_reduce, 2 * 8 * (g - 1) / g);  // comm.cpp:518: one double's worth
  if (g == 1) return local;
  auto parts = exchange_host(ctx, group, local.limbs().data(), sizeof(uint64_t) * ExactSum::kLimbs);
  ExactSum total;
  for (const auto& p : parts) {
    std::array<uint64_t, ExactSum::kLimbs> l{};
    std::memcpy(l.data(), p.data(), sizeof(l));
    total.merge(ExactSum::from_limbs(l));
  }
  return total;
}

int64_t all_reduce_count(RankCtx& ctx, const CommGroup& group, int64_t n) {
  const int g = group.size();
  ctx.count(Primitive::all_reduce, 2 * 8 * (g - 1) / g);  // comm.cpp:507
  if (g == 1) return n;
  int64_t total = 0;
  for (const auto& p : exchange_host(ctx, group, &n, sizeof(n))) {
    int64_t v;
    std::memcpy(&v, p.data(), sizeof(v));
    total += v;
  }
  return total;
}

namespace {
// balanced pairwise sum over [lo, hi) (tree_sum_into, comm.cpp:323-337)
void tree_sum(const std::vector<std::vector<double>>& parts, int lo, int hi, std::vector<double>& out) {
  if (hi - lo == 1) {
    out = parts[static_cast<size_t>(lo)];
    return;
  }
  const int mid = lo + (hi - lo) / 2;
  std::vector<double> a, b;
  tree_sum(parts, lo, mid, a);
  tree_sum(parts, mid, hi, b);
  out.resize(a.size());
  for (size_t i = 0; i < a.size(); ++i) out[i] = a[i] + b[i];
}
}  // namespace

std::vector<double> all_reduce_values(RankCtx& ctx, const CommGroup& group, const std::vector<double>& vals) {
  const int g = group.size();
  ctx.count(Primitive::all_reduce, 2 * static_cast<int64_t>(vals.size()) * 8 * (g - 1) / g);  // comm.cpp:343-344
  if (g == 1) return vals;
  auto raw = exchange_host(ctx, group, vals.data(), vals.size() * sizeof(double));
  std::vector<std::vector<double>> parts(static_cast<size_t>(g), std::vector<double>(vals.size()));
  for (int j = 0; j < g; ++j) std::memcpy(parts[static_cast<size_t>(j)].data(), raw[static_cast<size_t>(j)].data(),
                                          vals.size() * sizeof(double));
  std::vector<double> out;
  tree_sum(parts, 0, g, out);
  return out;
}

}  // namespace seqpar
