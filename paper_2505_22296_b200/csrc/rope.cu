// Rotary position embedding with GLOBAL position ids (rope_apply, reference
// proj/src/tensor.cpp:548-607; the global-id requirement is model.cpp:313-318, the paper's
// §5.2 pitfall), fused into the sequence->head row copies of the Ulysses all-to-all.
//
// Half-dim pairing as the reference: for head column j < dim/2,
//   lo' = lo*cos(p*theta_j) - hi*sin(p*theta_j),  hi' = lo*sin(p*theta_j) + hi*cos(p*theta_j)
// with theta_j = base^(-2j/dim) (tensor.cpp:559-562) and p the token's global position id.
// The backward is the inverse rotation (tensor.cpp:589-600): sign = -1.
//
// The angle table float2(cos, sin)[rows][dim/2] is built once per forward from the rank's
// position ids (angles in fp64, as the reference computes them) and reused by q, k and the
// backward's dq, dk; at c2 (L=32768, d=128) it is 16 MB and stays L2-resident while the copy
// kernels stream q/k through HBM. Copy kernels are HBM-bound: 2 x payload bytes + table reads
// (L2 hits shared by all heads of a row).
#include "common.cuh"

namespace spattn {
namespace {

__global__ void rope_table_kernel(float2* table, const int64_t* pos, int64_t rows, int half,
                                  int dim, double base) {
  const int64_t n = rows * half;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / half;
    const int j = (int)(i % half);
    const double theta = pow(base, -2.0 * (double)j / (double)dim);
    double s, c;
    sincos((double)pos[r] * theta, &s, &c);
    table[i] = make_float2((float)c, (float)s);
  }
}

struct RopeLaunch {
  CopyTaskSet ts;
  int64_t row_prefix[kMaxCopyTasks + 1];
};

__device__ __forceinline__ void rot(float lo, float hi, float2 cs, float sign, float& olo, float& ohi) {
  const float s = sign * cs.y;
  olo = fmaf(lo, cs.x, -hi * s);
  ohi = fmaf(lo, s, hi * cs.x);
}

// One warp per (task, row). VEC: lanes own (lo, hi) pairs of 8-element (16-byte) vectors of one
// head; else single element pairs. In-place (src == dst) is safe: each pair is read and written
// by the same thread.
template <bool VEC>
__global__ void __launch_bounds__(256) copy_rows_rope_kernel(RopeLaunch L) {
  const int64_t total = L.row_prefix[L.ts.n];
  const int lane = threadIdx.x % 32;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
  for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32; w < total; w += warps) {
    int ti = 0;
    while (ti + 1 < L.ts.n && L.row_prefix[ti + 1] <= w) ++ti;
    const CopyTask& T = L.ts.t[ti];
    const int64_t r = w - L.row_prefix[ti];
    const __nv_bfloat16* src =
        reinterpret_cast<const __nv_bfloat16*>(T.src) + (T.src_row0 + r) * T.src_row_stride + T.src_col0;
    __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(T.dst) + (T.dst_row0 + r) * T.dst_row_stride + T.dst_col0;
    const int dim = T.rope_dim, half = dim / 2;
    const float sign = (float)T.rope_sign;
    const float2* tb = T.rope + ((T.rope_row0 + r) % T.rope_mod) * half;
    if (VEC) {
      const int per_head = dim / 16;
      const int64_t np = T.cols / 16;
      for (int64_t p = lane; p < np; p += 32) {
        const int64_t h = p / per_head;
        const int jv = (int)(p % per_head) * 8;
        const int64_t off = h * dim + jv;
        const uint4 a = *reinterpret_cast<const uint4*>(src + off);
        const uint4 b = *reinterpret_cast<const uint4*>(src + off + half);
        const float4* t4 = reinterpret_cast<const float4*>(tb + jv);
        const uint32_t av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
        uint32_t oa[4], ob[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float4 cs = __ldg(t4 + q);  // (cos, sin) of columns jv+2q, jv+2q+1
          const float2 lo = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&av[q]));
          const float2 hi = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&bv[q]));
          float l0, h0, l1, h1;
          rot(lo.x, hi.x, make_float2(cs.x, cs.y), sign, l0, h0);
          rot(lo.y, hi.y, make_float2(cs.z, cs.w), sign, l1, h1);
          oa[q] = pack_bf16(l0, l1);
          ob[q] = pack_bf16(h0, h1);
        }
        *reinterpret_cast<uint4*>(dst + off) = make_uint4(oa[0], oa[1], oa[2], oa[3]);
        *reinterpret_cast<uint4*>(dst + off + half) = make_uint4(ob[0], ob[1], ob[2], ob[3]);
      }
    } else {
      const int64_t np = T.cols / 2;
      for (int64_t p = lane; p < np; p += 32) {
        const int64_t h = p / half;
        const int j = (int)(p % half);
        const int64_t off = h * dim + j;
        float lo = __bfloat162float(src[off]), hi = __bfloat162float(src[off + half]), olo, ohi;
        rot(lo, hi, tb[j], sign, olo, ohi);
        dst[off] = __float2bfloat16_rn(olo);
        dst[off + half] = __float2bfloat16_rn(ohi);
      }
    }
    for (int64_t i = lane; i < T.zero_cols; i += 32) dst[T.cols + i] = __float2bfloat16_rn(0.f);
  }
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

void launch_rope_table(float2* table, const int64_t* dpos, int64_t rows, int dim, double base,
                       cudaStream_t s) {
  const int64_t n = rows * (dim / 2);
  if (n == 0) return;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  rope_table_kernel<<<(int)blocks, 256, 0, s>>>(table, dpos, rows, dim / 2, dim, base);
  note_launch();
}

void launch_copy_tasks_rope(const CopyTaskSet& ts, cudaStream_t s) {
  RopeLaunch L;
  L.ts = ts;
  L.row_prefix[0] = 0;
  bool vec = true;
  for (int i = 0; i < ts.n; ++i) {
    const CopyTask& t = ts.t[i];
    L.row_prefix[i + 1] = L.row_prefix[i] + t.rows;
    int64_t a = 16;
    for (int64_t v : {(int64_t)reinterpret_cast<uintptr_t>(t.src), (int64_t)reinterpret_cast<uintptr_t>(t.dst),
                      t.src_row_stride * 2, t.dst_row_stride * 2, t.src_col0 * 2, t.dst_col0 * 2})
      a = gcd64(a, v == 0 ? 16 : v);
    vec = vec && a == 16 && t.rope_dim % 16 == 0;
  }
  const int64_t total = L.row_prefix[ts.n];
  if (total == 0) return;
  int64_t blocks = (total + 7) / 8;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (vec)
    copy_rows_rope_kernel<true><<<(int)blocks, 256, 0, s>>>(L);
  else
    copy_rows_rope_kernel<false><<<(int)blocks, 256, 0, s>>>(L);
  note_launch();
}

}  // namespace spattn
