// HBM-bound data-movement kernels of the SP layer:
//   * the fused pack/pad -> exchange -> unpack/unpad row copier used by every all-to-all
//     (all_to_all_values + copy_region, comm.cpp:247-321; pad_axis_zeros / slice_axis,
//     tensor.cpp:360-416), the zigzag/naive row permutation (shard_rows / gather_rows,
//     partition.cpp:124-158) and the ring KV rotation (ring_shift, comm.cpp:449-460);
//   * the LSE merge (merge_piece, attention.cpp:117-149);
//   * fp32 <-> bf16 conversions for gradient accumulators.
// All copies are byte-exact (dtype-agnostic, 16-byte vectorised when alignment allows).
#include <algorithm>
#include <atomic>
#include <cstdlib>

#include "tc.cuh"

namespace spattn {
namespace {

struct CopyLaunch {
  CopyTaskSet ts;
  int64_t row_prefix[kMaxCopyTasks + 1];
};

template <int VW>
struct Vec;
template <>
struct Vec<16> { using T = uint4; };
template <>
struct Vec<8> { using T = uint2; };
template <>
struct Vec<4> { using T = uint32_t; };
template <>
struct Vec<2> { using T = uint16_t; };
template <>
struct Vec<1> { using T = uint8_t; };

// One warp per chunk of up to `rpc` consecutive rows of one task (chunk_prefix counts chunks per
// task). The chunk's rows x (cols + zero_cols) vectors are flattened and each lane keeps four
// independent 16-byte (or narrower) loads in flight before their stores, whatever the row
// length: the all-to-all packs move rows of a few hundred bytes to a few KB, where one row per
// warp leaves the memory system starved.
template <int VW>
__global__ void __launch_bounds__(256) copy_rows_kernel(CopyLaunch L, int elem_bytes, int rpc) {
  using V = typename Vec<VW>::T;
  const int64_t total = L.row_prefix[L.ts.n];  // chunks
  const int lane = threadIdx.x % 32;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
  for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32; w < total; w += warps) {
    int lo = 0, hi = L.ts.n - 1;  // the task of chunk w
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (L.row_prefix[mid + 1] > w) hi = mid; else lo = mid + 1;
    }
    const CopyTask& T = L.ts.t[lo];
    const int64_t r0 = (w - L.row_prefix[lo]) * rpc;
    const int64_t nr = min((int64_t)rpc, T.rows - r0);
    const int64_t nv = T.cols * elem_bytes / VW, nz = T.zero_cols * elem_bytes / VW, rv = nv + nz;
    const uint8_t* src = reinterpret_cast<const uint8_t*>(T.src) +
                         ((T.src_row0 + r0) * T.src_row_stride + T.src_col0) * elem_bytes;
    uint8_t* dst = reinterpret_cast<uint8_t*>(T.dst) + ((T.dst_row0 + r0) * T.dst_row_stride + T.dst_col0) * elem_bytes;
    const int64_t ss = T.src_row_stride * elem_bytes, ds = T.dst_row_stride * elem_bytes;
    const int64_t n = nr * rv;
    V z;
    memset(&z, 0, sizeof(V));
    for (int64_t i = lane; i < n; i += 128) {
      V x[4];
      int64_t off[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int64_t e = i + 32 * k;
        const int r = (int)e / (int)rv;  // chunk extents fit 32 bits
        const int64_t c = e - (int64_t)r * rv;
        off[k] = e < n ? r * ds + c * VW : -1;
        x[k] = (e < n && c < nv) ? *reinterpret_cast<const V*>(src + r * ss + c * VW) : z;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (off[k] >= 0) *reinterpret_cast<V*>(dst + off[k]) = x[k];
    }
  }
}

// ----------------------------------------------------------- TMA-staged row copier
// Plain row copies (every all-to-all pack / unpack without padding or RoPE, shard / gather
// rows, ring payloads) move as 2-D TMA boxes: per task a source and a destination tensor map
// over its rows (8-byte elements, no swizzle), boxes of up to 256 x 2 KB (32 KB) staged through
// shared memory — TMA load into a slot, TMA store out of it — by one issuing lane per CTA with
// several loads and stores in flight (TmaLaunch::slots / ahead). A box covers many rows, so the
// ~1 KB rows of an SP=8 pack no longer cost one copy operation each.
#ifndef SPATTN_TMA_TASKS
#define SPATTN_TMA_TASKS 48
#endif
constexpr int kTmaTasks = SPATTN_TMA_TASKS;  // 2 maps + scalars per task in the 32 KB parameter space
// Shared memory: kTmaStage bytes split into slots of one box each (32 KB boxes: 7 slots, 4 loads
// ahead; the kernel takes the slot geometry as a launch parameter).
constexpr int kTmaMaxSlots = 28, kTmaStage = 7 * 32768;
constexpr int kTmaSmem = kTmaStage + kTmaMaxSlots * 8;
struct TmaTask {
  CUtensorMap src, dst;
  int br, ncb;  // box rows, column boxes per row block
};
struct TmaLaunch {
  TmaTask t[kTmaTasks];
  int64_t unit_prefix[kTmaTasks + 1];  // cumulative row blocks x column boxes
  int box_bytes[kTmaTasks];            // bytes one full box moves (expect_tx; OOB parts count too)
  int n;
  int slots, ahead, slot_bytes;
};
static_assert(sizeof(TmaLaunch) <= 32000, "kernel parameter space");

__global__ void __launch_bounds__(32, 1) copy_rows_tma_kernel(const __grid_constant__ TmaLaunch L) {
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t slots = smem_u32(smem), bars = slots + kTmaStage;
  if (threadIdx.x != 0) return;
  const int NS = L.slots, NA = L.ahead, SB = L.slot_bytes;
  for (int i = 0; i < NS; ++i) tc::mbar_init(bars + 8 * i, 1);
  tc::fence_barrier_init();
  const int64_t total = L.unit_prefix[L.n];
  const int64_t per = (total + gridDim.x - 1) / gridDim.x;
  const int64_t u0 = min(total, (int64_t)blockIdx.x * per), u1 = min(total, u0 + per);
  const int64_t n = u1 - u0;
  if (n <= 0) return;
  int tl = 0, ts = 0;  // task cursors of the load and store walks (units only move forward)
  auto locate = [&](int64_t u, int& t, int& x, int& y) {
    while (t + 1 < L.n && L.unit_prefix[t + 1] <= u) ++t;
    const int64_t k = u - L.unit_prefix[t];
    x = (int)(k % L.t[t].ncb) * 256;
    y = (int)(k / L.t[t].ncb) * L.t[t].br;
  };
  auto load = [&](int64_t j) {
    int x, y;
    locate(u0 + j, tl, x, y);
    const int sl = (int)(j % NS);
    tc::mbar_expect_tx(bars + 8 * sl, (uint32_t)L.box_bytes[tl]);
    tc::tma_load_2d(slots + sl * SB, &L.t[tl].src, x, y, bars + 8 * sl);
  };
  for (int64_t j = 0; j < n && j < NA; ++j) load(j);
  for (int64_t j = 0; j < n; ++j) {
    const int sl = (int)(j % NS);
    int x, y;
    locate(u0 + j, ts, x, y);
    tc::mbar_wait(bars + 8 * sl, (uint32_t)((j / NS) & 1));
    tc::tma_store_2d(&L.t[ts].dst, slots + sl * SB, x, y);
    tc::bulk_commit();
    if (j + NA < n) {
      // the store that last used slot (j + NA) % NS, j + NA - NS, has read it once at most
      // NS - NA later stores are pending
      switch (NS - NA) {
        case 12: tc::bulk_wait_read<12>(); break;
        case 6: tc::bulk_wait_read<6>(); break;
        case 3: tc::bulk_wait_read<3>(); break;
        default: tc::bulk_wait_read<0>(); break;
      }
      load(j + NA);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");  // stores complete before exit
}

// fp32 variant that accumulates: dst += src (the repeat_heads backward group sum,
// tensor.cpp:437-447, when kv windows of different ranks share a head).
__global__ void __launch_bounds__(256) add_rows_kernel(CopyLaunch L) {
  const int64_t total = L.row_prefix[L.ts.n];
  const int lane = threadIdx.x % 32;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
  for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32; w < total; w += warps) {
    int ti = 0;
    while (ti + 1 < L.ts.n && L.row_prefix[ti + 1] <= w) ++ti;
    const CopyTask& T = L.ts.t[ti];
    const int64_t r = w - L.row_prefix[ti];
    const float* src = reinterpret_cast<const float*>(T.src) + (T.src_row0 + r) * T.src_row_stride + T.src_col0;
    float* dst = reinterpret_cast<float*>(T.dst) + (T.dst_row0 + r) * T.dst_row_stride + T.dst_col0;
    for (int64_t i = lane; i < T.cols; i += 32) dst[i] += src[i];
  }
}

__global__ void lse_merge_kernel(float* acc_o, float* acc_lse, const float* o, const float* lse,
                                 int64_t rows, int d) {
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x % 32;
  if (row >= rows) return;
  const float la = acc_lse[row], lb = lse[row];
  const float mx = fmaxf(la, lb);
  if (lb == -INFINITY) return;  // empty piece: acc unchanged (attention.cpp:130-134)
  float wa, wb, ln;
  if (la == -INFINITY) {  // empty accumulator adopts the piece (attention.cpp:118-121)
    wa = 0.f, wb = 1.f, ln = lb;
  } else {
    ln = mx + log1pf(__expf(fminf(la, lb) - mx));
    wa = __expf(la - ln);
    wb = __expf(lb - ln);
  }
  float* ap = acc_o + row * d;
  const float* bp = o + row * d;
  for (int i = lane; i < d; i += 32) ap[i] = la == -INFINITY ? bp[i] : ap[i] * wa + bp[i] * wb;
  __syncwarp();
  if (lane == 0) acc_lse[row] = ln;
}

__global__ void fill_f32_kernel(float* p, float v, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

__global__ void f32_to_bf16_2d_kernel(__nv_bfloat16* dst, int64_t dst_stride, const float* src,
                                      int64_t src_stride, int64_t rows, int64_t cols, float scale) {
  const int64_t n = rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / cols, c = i % cols;
    dst[r * dst_stride + c] = __float2bfloat16_rn(src[r * src_stride + c] * scale);
  }
}

__global__ void f32_to_bf16_kernel(__nv_bfloat162* dst, const float2* src, float scale, int64_t n2) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float2 v = src[i];
    dst[i] = __floats2bfloat162_rn(v.x * scale, v.y * scale);
  }
}

// 8 values per thread: two 16-byte loads, one 16-byte store, unrolled twice so four loads are
// in flight per thread (the 8-byte grid-stride loop above reaches ~77 % of the HBM rate)
__global__ void __launch_bounds__(256) f32_to_bf16_v8_kernel(uint4* dst, const float4* src, float scale, int64_t n8) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  auto cvt = [&](const float4& a, const float4& b) {
    __nv_bfloat162 p0 = __floats2bfloat162_rn(a.x * scale, a.y * scale);
    __nv_bfloat162 p1 = __floats2bfloat162_rn(a.z * scale, a.w * scale);
    __nv_bfloat162 p2 = __floats2bfloat162_rn(b.x * scale, b.y * scale);
    __nv_bfloat162 p3 = __floats2bfloat162_rn(b.z * scale, b.w * scale);
    return make_uint4(*reinterpret_cast<uint32_t*>(&p0), *reinterpret_cast<uint32_t*>(&p1),
                      *reinterpret_cast<uint32_t*>(&p2), *reinterpret_cast<uint32_t*>(&p3));
  };
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; i + stride < n8; i += 2 * stride) {
    const float4 a0 = __ldcs(src + 2 * i), b0 = __ldcs(src + 2 * i + 1);
    const float4 a1 = __ldcs(src + 2 * (i + stride)), b1 = __ldcs(src + 2 * (i + stride) + 1);
    dst[i] = cvt(a0, b0);
    dst[i + stride] = cvt(a1, b1);
  }
  if (i < n8) dst[i] = cvt(__ldcs(src + 2 * i), __ldcs(src + 2 * i + 1));
}

__global__ void bf16_to_f32_kernel(float* dst, const __nv_bfloat16* src, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = __bfloat162float(src[i]);
}

__global__ void f32_add_2d_kernel(float* dst, int64_t dst_stride, const float* src,
                                  int64_t src_stride, int64_t rows, int64_t cols) {
  const int64_t n = rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / cols, c = i % cols;
    dst[r * dst_stride + c] += src[r * src_stride + c];
  }
}

int grid_for(int64_t n, int per_block) {
  int64_t b = (n + per_block - 1) / per_block;
  const int64_t cap = 148 * 16;
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

int64_t gcd64(int64_t a, int64_t b) {
  while (b) {
    const int64_t t = a % b;
    a = b;
    b = t;
  }
  return a < 0 ? -a : a;
}

}  // namespace

namespace {
std::atomic<long long> g_launches{0};
}
void note_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
long long launch_count() { return g_launches.load(std::memory_order_relaxed); }

// TMA path for a task set: every row run 16-byte aligned with a 16-byte-multiple width, no
// padding columns, at most kTmaTasks tasks; false = use the warp copier. Tasks may carry their
// own element size (CopyTask::elem), so moves of different dtypes share one launch.
bool launch_copy_tasks_tma(const CopyTaskSet& ts, int elem_bytes, cudaStream_t s) {
  if (ts.n > kTmaTasks) return false;
  TmaLaunch L;
  L.n = ts.n;
  L.unit_prefix[0] = 0;
  int64_t bytes = 0;
  for (int i = 0; i < ts.n; ++i) {
    const CopyTask& t = ts.t[i];
    const int64_t eb = t.elem ? t.elem : elem_bytes;
    if (t.zero_cols || t.cols <= 0 || (t.cols * eb) % 16 || t.rows <= 0 || t.rows > (int64_t)1 << 31) return false;
    bytes += t.rows * t.cols * eb;
  }
  // box size: 32 KB (smaller boxes measured slower even for 16 MB launches of 256-byte rows:
  // the TMA unit's cost follows the rows, not the boxes; profiles/r2/copy_kernels.md)
  constexpr int box = 32768;
  L.slot_bytes = box;
  L.slots = std::min(kTmaMaxSlots, kTmaStage / box);
  L.ahead = std::max(1, L.slots * 4 / 7);
  for (int i = 0; i < ts.n; ++i) {
    const CopyTask& t = ts.t[i];
    const int64_t eb = t.elem ? t.elem : elem_bytes;
    const int64_t rb = t.cols * eb;
    const char* src = static_cast<const char*>(t.src) + (t.src_row0 * t.src_row_stride + t.src_col0) * eb;
    char* dst = static_cast<char*>(t.dst) + (t.dst_row0 * t.dst_row_stride + t.dst_col0) * eb;
    if (reinterpret_cast<uintptr_t>(src) % 16 || reinterpret_cast<uintptr_t>(dst) % 16 ||
        (t.src_row_stride * eb) % 16 || (t.dst_row_stride * eb) % 16)
      return false;
    const int64_t w8 = rb / 8, bw = std::min<int64_t>(256, w8);
    const int br = (int)std::max<int64_t>(1, std::min<int64_t>(256, box / (bw * 8)));
    if (!make_tma_rows_u64(&L.t[i].src, src, w8, t.rows, t.src_row_stride * eb, (uint32_t)bw, br) ||
        !make_tma_rows_u64(&L.t[i].dst, dst, w8, t.rows, t.dst_row_stride * eb, (uint32_t)bw, br))
      return false;
    L.t[i].br = br;
    L.t[i].ncb = (int)((w8 + 255) / 256);
    L.box_bytes[i] = (int)(bw * 8 * br);
    L.unit_prefix[i + 1] = L.unit_prefix[i] + ((t.rows + br - 1) / br) * L.t[i].ncb;
  }
  const int64_t total = L.unit_prefix[ts.n];
  if (total == 0) return true;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(148, total));
  ensure_smem_for(copy_rows_tma_kernel, kTmaSmem);
  copy_rows_tma_kernel<<<grid, 32, kTmaSmem, s>>>(L);
  note_launch();
  return true;
}

void launch_copy_tasks(const CopyTaskSet& ts, int elem_bytes, cudaStream_t s) {
  if (ts.n > 0 && ts.t[0].rope) return launch_copy_tasks_rope(ts, s);
  static const bool no_tma = getenv("SPATTN_NO_TMA_COPY") != nullptr;  // A/B switch (same bytes)
  if (!no_tma && launch_copy_tasks_tma(ts, elem_bytes, s)) return;
  bool mixed = false;
  for (int i = 0; i < ts.n; ++i) mixed |= ts.t[i].elem != 0 && ts.t[i].elem != elem_bytes;
  if (mixed) {  // the warp copier takes one element size per launch: one launch per size
    for (int i = 0; i < ts.n; ++i) {
      const int e = ts.t[i].elem ? ts.t[i].elem : elem_bytes;
      bool first = true;
      for (int j = 0; j < i; ++j) first &= (ts.t[j].elem ? ts.t[j].elem : elem_bytes) != e;
      if (!first) continue;
      CopyTaskSet sub{};
      for (int j = 0; j < ts.n; ++j)
        if ((ts.t[j].elem ? ts.t[j].elem : elem_bytes) == e) {
          sub.t[sub.n] = ts.t[j];
          sub.t[sub.n++].elem = 0;
        }
      launch_copy_tasks(sub, e, s);
    }
    return;
  }
  CopyLaunch L;
  L.ts = ts;
  L.row_prefix[0] = 0;
  int64_t align = 16, bytes = 0, rows = 0;
  for (int i = 0; i < ts.n; ++i) {
    bytes += ts.t[i].rows * (ts.t[i].cols + ts.t[i].zero_cols) * elem_bytes;
    rows += ts.t[i].rows;
  }
  // rows per warp chunk: about 4 KB per chunk
  constexpr int chunk_bytes = 4096;  // measured best of 1 row / 4 KB / 16 KB per warp (profiles/r2/copy_kernels.md)
  const int rpc = (int)std::max<int64_t>(1, chunk_bytes / std::max<int64_t>(1, rows ? bytes / rows : 1));
  for (int i = 0; i < ts.n; ++i) {
    const CopyTask& t = ts.t[i];
    L.row_prefix[i + 1] = L.row_prefix[i] + (t.rows + rpc - 1) / rpc;
    for (int64_t v : {(int64_t)reinterpret_cast<uintptr_t>(t.src), (int64_t)reinterpret_cast<uintptr_t>(t.dst),
                      t.src_row_stride * elem_bytes, t.dst_row_stride * elem_bytes,
                      (t.src_row0 * t.src_row_stride + t.src_col0) * elem_bytes,
                      (t.dst_row0 * t.dst_row_stride + t.dst_col0) * elem_bytes, t.cols * elem_bytes,
                      t.zero_cols * elem_bytes})
      align = gcd64(align, v == 0 ? 16 : v);
  }
  const int64_t total = L.row_prefix[ts.n];
  if (total == 0) return;
  const int grid = grid_for(total, 8);
  switch (align) {
    case 16: copy_rows_kernel<16><<<grid, 256, 0, s>>>(L, elem_bytes, rpc); break;
    case 8: copy_rows_kernel<8><<<grid, 256, 0, s>>>(L, elem_bytes, rpc); break;
    case 4: copy_rows_kernel<4><<<grid, 256, 0, s>>>(L, elem_bytes, rpc); break;
    case 2: copy_rows_kernel<2><<<grid, 256, 0, s>>>(L, elem_bytes, rpc); break;
    default: copy_rows_kernel<1><<<grid, 256, 0, s>>>(L, elem_bytes, rpc); break;
  }
  note_launch();
}

void launch_add_tasks_f32(const CopyTaskSet& ts, cudaStream_t s) {
  CopyLaunch L;
  L.ts = ts;
  L.row_prefix[0] = 0;
  for (int i = 0; i < ts.n; ++i) L.row_prefix[i + 1] = L.row_prefix[i] + ts.t[i].rows;
  const int64_t total = L.row_prefix[ts.n];
  if (total == 0) return;
  add_rows_kernel<<<grid_for(total, 8), 256, 0, s>>>(L);
  note_launch();
}

void launch_lse_merge(float* acc_o, float* acc_lse, const float* o, const float* lse, int64_t rows,
                      int d, cudaStream_t s) {
  if (rows == 0) return;
  lse_merge_kernel<<<(int)((rows + 7) / 8), 256, 0, s>>>(acc_o, acc_lse, o, lse, rows, d);
  note_launch();
}

void launch_fill_f32(float* p, float v, int64_t n, cudaStream_t s) {
  if (n == 0) return;
  fill_f32_kernel<<<grid_for(n, 1024), 256, 0, s>>>(p, v, n);
  note_launch();
}

void launch_f32_to_bf16(void* dst, const float* src, float scale, int64_t n, cudaStream_t s) {
  if (n == 0) return;
  if (n % 8 == 0 && reinterpret_cast<uintptr_t>(dst) % 16 == 0 && reinterpret_cast<uintptr_t>(src) % 16 == 0) {
    f32_to_bf16_v8_kernel<<<grid_for(n / 8, 512), 256, 0, s>>>(reinterpret_cast<uint4*>(dst),
                                                               reinterpret_cast<const float4*>(src), scale, n / 8);
    note_launch();
  } else if (n % 2 == 0) {
    f32_to_bf16_kernel<<<grid_for(n / 2, 1024), 256, 0, s>>>(
        reinterpret_cast<__nv_bfloat162*>(dst), reinterpret_cast<const float2*>(src), scale, n / 2);
  note_launch();
  } else {
    f32_to_bf16_2d_kernel<<<grid_for(n, 1024), 256, 0, s>>>(reinterpret_cast<__nv_bfloat16*>(dst),
                                                            n, src, n, 1, n, scale);
  note_launch();
  }
}

void launch_bf16_to_f32(float* dst, const void* src, int64_t n, cudaStream_t s) {
  if (n == 0) return;
  bf16_to_f32_kernel<<<grid_for(n, 1024), 256, 0, s>>>(
      dst, reinterpret_cast<const __nv_bfloat16*>(src), n);
  note_launch();
}

void launch_f32_to_bf16_2d(void* dst, int64_t dst_stride, const float* src, int64_t src_stride,
                           int64_t rows, int64_t cols, float scale, cudaStream_t s) {
  if (rows * cols == 0) return;
  f32_to_bf16_2d_kernel<<<grid_for(rows * cols, 1024), 256, 0, s>>>(
      reinterpret_cast<__nv_bfloat16*>(dst), dst_stride, src, src_stride, rows, cols, scale);
  note_launch();
}

__global__ void __launch_bounds__(256) f32_add_v4_kernel(float4* dst, const float4* src, int64_t n4) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    float4 a = dst[i];
    const float4 b = src[i];
    a.x += b.x, a.y += b.y, a.z += b.z, a.w += b.w;
    dst[i] = a;
  }
}

void launch_f32_add(float* dst, const float* src, int64_t n, cudaStream_t s) {
  if (n == 0) return;
  if (n % 4 == 0 && reinterpret_cast<uintptr_t>(dst) % 16 == 0 && reinterpret_cast<uintptr_t>(src) % 16 == 0) {
    f32_add_v4_kernel<<<grid_for(n / 4, 512), 256, 0, s>>>(reinterpret_cast<float4*>(dst),
                                                           reinterpret_cast<const float4*>(src), n / 4);
    note_launch();
  } else {
    launch_f32_add_2d(dst, n, src, n, 1, n, s);
  }
}

void launch_f32_add_2d(float* dst, int64_t dst_stride, const float* src, int64_t src_stride,
                       int64_t rows, int64_t cols, cudaStream_t s) {
  if (rows * cols == 0) return;
  f32_add_2d_kernel<<<grid_for(rows * cols, 1024), 256, 0, s>>>(dst, dst_stride, src, src_stride,
                                                                rows, cols);
  note_launch();
}

}  // namespace spattn
