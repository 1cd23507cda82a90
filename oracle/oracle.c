/* TEST INFRASTRUCTURE ONLY — see oracle.h. Plain-C restatement of the reference's f64
 * attention block math (/root/reference/proj/src/attention.cpp:61-216) and its fixture RNG
 * (/root/reference/proj/src/tensor.cpp:724-739). OpenMP only splits independent rows/heads;
 * the per-row arithmetic order is the reference's. */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

uint64_t orc_rng_next(uint64_t* state) {
  /* tensor.hpp:162 — a zero seed is replaced by the golden-ratio constant */
  if (*state == 0) *state = 0x9e3779b97f4a7c15ull;
  *state += 0x9e3779b97f4a7c15ull; /* tensor.cpp:727 */
  uint64_t z = *state;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

void orc_rng_fill_uniform(uint64_t* state, double lo, double hi, double* out, int64_t n) {
  for (int64_t i = 0; i < n; ++i) {
    const double u = (double)(orc_rng_next(state) >> 11) * 0x1.0p-53; /* tensor.cpp:735-737 */
    out[i] = lo + (hi - lo) * u;                                      /* tensor.cpp:739 */
  }
}

static inline int admitted(int causal, const int64_t* qpos, const int64_t* qseg,
                           const int64_t* kpos, const int64_t* kseg, int64_t i, int64_t j) {
  if (causal && kpos[j] > qpos[i]) return 0; /* attention.cpp:89 */
  if (qseg && kseg && qseg[i] != kseg[j]) return 0;
  return 1;
}

int64_t orc_attn_block_forward(int64_t bs, int64_t heads, int64_t kv_heads, int64_t dim,
                               const double* q, const int64_t* qpos, const int64_t* qseg,
                               int64_t lq, const double* k, const double* v,
                               const int64_t* kpos, const int64_t* kseg, int64_t lk,
                               int causal, double scale, double* numerator, double* row_max,
                               double* row_norm) {
  const int64_t rep = heads / kv_heads;
  const int64_t rows = bs * lq * heads;
  int64_t pairs = 0;
  memset(numerator, 0, sizeof(double) * (size_t)(rows * dim));
#pragma omp parallel reduction(+ : pairs)
  {
    double* scores = (double*)malloc(sizeof(double) * (size_t)(lk > 0 ? lk : 1));
#pragma omp for schedule(dynamic, 16)
    for (int64_t row = 0; row < rows; ++row) {
      const int64_t h = row % heads, i = (row / heads) % lq, b = row / (heads * lq);
      const int64_t hk = h / rep;
      const double* qrow = q + row * dim;
      double m = -INFINITY;
      for (int64_t j = 0; j < lk; ++j) { /* attention.cpp:86-97 */
        if (!admitted(causal, qpos, qseg, kpos, kseg, i, j)) continue;
        const double* krow = k + ((b * lk + j) * kv_heads + hk) * dim;
        double dot = 0.0;
        for (int64_t c = 0; c < dim; ++c) dot += qrow[c] * krow[c];
        scores[j] = dot * scale;
        if (scores[j] > m) m = scores[j];
        ++pairs;
      }
      row_max[row] = -INFINITY;
      row_norm[row] = 0.0;
      if (m == -INFINITY) continue; /* :98 nothing admitted */
      double* num = numerator + row * dim;
      double norm = 0.0;
      for (int64_t j = 0; j < lk; ++j) { /* :101-107 */
        if (!admitted(causal, qpos, qseg, kpos, kseg, i, j)) continue;
        const double w = exp(scores[j] - m);
        norm += w;
        const double* vrow = v + ((b * lk + j) * kv_heads + hk) * dim;
        for (int64_t c = 0; c < dim; ++c) num[c] += w * vrow[c];
      }
      row_max[row] = m;
      row_norm[row] = norm;
    }
    free(scores);
  }
  return pairs;
}

void orc_merge_piece(int64_t rows, int64_t dim, int acc_empty, double* acc_num, double* acc_max,
                     double* acc_norm, const double* num, const double* mx, const double* norm) {
  if (acc_empty) { /* attention.cpp:118-121 */
    memcpy(acc_num, num, sizeof(double) * (size_t)(rows * dim));
    memcpy(acc_max, mx, sizeof(double) * (size_t)rows);
    memcpy(acc_norm, norm, sizeof(double) * (size_t)rows);
    return;
  }
  for (int64_t row = 0; row < rows; ++row) {
    const double mb = mx[row];
    if (mb == -INFINITY) continue; /* :130 */
    const double ma = acc_max[row];
    double* na = acc_num + row * dim;
    const double* nb = num + row * dim;
    if (ma == -INFINITY) { /* :133-139 adopt */
      acc_max[row] = mb;
      acc_norm[row] = norm[row];
      memcpy(na, nb, sizeof(double) * (size_t)dim);
      continue;
    }
    const double m = ma > mb ? ma : mb; /* :140-147 */
    const double ca = exp(ma - m), cb = exp(mb - m);
    acc_max[row] = m;
    acc_norm[row] = acc_norm[row] * ca + norm[row] * cb;
    for (int64_t c = 0; c < dim; ++c) na[c] = na[c] * ca + nb[c] * cb;
  }
}

void orc_finalize_piece(int64_t rows, int64_t dim, const double* num, const double* mx,
                        const double* norm, double* out, double* lse) {
  for (int64_t row = 0; row < rows; ++row) { /* attention.cpp:151-165 */
    double* o = out + row * dim;
    if (norm[row] <= 0.0) {
      memset(o, 0, sizeof(double) * (size_t)dim);
      lse[row] = -INFINITY;
      continue;
    }
    const double inv = 1.0 / norm[row];
    for (int64_t c = 0; c < dim; ++c) o[c] = num[row * dim + c] * inv;
    lse[row] = mx[row] + log(norm[row]);
  }
}

int64_t orc_attn_block_backward(int64_t bs, int64_t heads, int64_t kv_heads, int64_t dim,
                                const double* q, const int64_t* qpos, const int64_t* qseg,
                                int64_t lq, const double* k, const double* v,
                                const int64_t* kpos, const int64_t* kseg, int64_t lk,
                                int causal, double scale, const double* out, const double* lse,
                                const double* dout, double* dq, double* dk, double* dv) {
  const int64_t rep = heads / kv_heads;
  int64_t pairs = 0;
  /* one task per (batch, kv head): dk/dv rows of that head are written by one thread only */
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : pairs)
  for (int64_t task = 0; task < bs * kv_heads; ++task) {
    const int64_t b = task / kv_heads, hk = task % kv_heads;
    for (int64_t i = 0; i < lq; ++i) {
      for (int64_t h = hk * rep; h < (hk + 1) * rep; ++h) {
        const int64_t row = (b * lq + i) * heads + h;
        if (lse[row] == -INFINITY) continue; /* attention.cpp:184 */
        const double* qrow = q + row * dim;
        const double* orow = out + row * dim;
        const double* dorow = dout + row * dim;
        double* dqrow = dq + row * dim;
        double delta = 0.0; /* :189-191 */
        for (int64_t c = 0; c < dim; ++c) delta += dorow[c] * orow[c];
        for (int64_t j = 0; j < lk; ++j) {
          if (!admitted(causal, qpos, qseg, kpos, kseg, i, j)) continue;
          const int64_t kidx = ((b * lk + j) * kv_heads + hk) * dim;
          const double* krow = k + kidx;
          const double* vrow = v + kidx;
          double dot = 0.0;
          for (int64_t c = 0; c < dim; ++c) dot += qrow[c] * krow[c];
          const double prob = exp(dot * scale - lse[row]); /* :198 */
          double dprob = 0.0;
          for (int64_t c = 0; c < dim; ++c) dprob += dorow[c] * vrow[c];
          const double dscore = prob * (dprob - delta) * scale; /* :201 */
          double* dkrow = dk + kidx;
          double* dvrow = dv + kidx;
          for (int64_t c = 0; c < dim; ++c) { /* :204-208 */
            dvrow[c] += prob * dorow[c];
            dqrow[c] += dscore * krow[c];
            dkrow[c] += dscore * qrow[c];
          }
          ++pairs;
        }
      }
    }
  }
  return pairs;
}
