/* TEST INFRASTRUCTURE ONLY — CPU restatement of the reference's f64 attention math.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load this.
 * The product library (paper_2505_22296_b200/csrc) never links or calls it.
 *
 * Every function cites the reference file:line it restates (paths relative to
 * /root/reference/proj). Layout/permutation/byte arithmetic lives in seqpar_oracle.py (numpy).
 */
#ifndef SPATTN_ORACLE_H
#define SPATTN_ORACLE_H
#include <stdint.h>

/* splitmix64 (tensor.cpp:724-733); state 0 is replaced as in tensor.hpp:162 */
uint64_t orc_rng_next(uint64_t* state);
/* uniform_range(lo, hi) draws (tensor.cpp:735-739), n of them, in order */
void orc_rng_fill_uniform(uint64_t* state, double lo, double hi, double* out, int64_t n);

/* attn_block_forward (attention.cpp:61-115), generalised two ways that keep its arithmetic:
 *   - k/v carry kv_heads heads; query head h reads kv head h / (heads / kv_heads), which is
 *     what repeat_heads (tensor.cpp:418-450) materialises before the reference engine runs;
 *   - optional segment ids (NULL = none) add "same document" to the admission test.
 * Outputs: numerator [bs,lq,heads,dim], row_max/row_norm [bs,lq,heads].
 * Returns the admitted pair count (the reference charges 4*dim flops per pair, :113). */
int64_t orc_attn_block_forward(int64_t bs, int64_t heads, int64_t kv_heads, int64_t dim,
                               const double* q, const int64_t* qpos, const int64_t* qseg,
                               int64_t lq, const double* k, const double* v,
                               const int64_t* kpos, const int64_t* kseg, int64_t lk,
                               int causal, double scale, double* numerator, double* row_max,
                               double* row_norm);

/* merge_piece (attention.cpp:117-149). acc_empty=1 adopts the piece bit-identically (:118-121). */
void orc_merge_piece(int64_t rows, int64_t dim, int acc_empty, double* acc_num, double* acc_max,
                     double* acc_norm, const double* num, const double* mx, const double* norm);

/* finalize_piece (attention.cpp:151-165): out = num / norm, lse = max + log(norm). */
void orc_finalize_piece(int64_t rows, int64_t dim, const double* num, const double* mx,
                        const double* norm, double* out, double* lse);

/* attn_block_backward (attention.cpp:167-216), += into dq [bs,lq,heads,dim] and
 * dk/dv [bs,lk,kv_heads,dim] (the group sum repeat_heads' backward does, tensor.cpp:437-447).
 * Returns admitted pairs (10*dim flops each, :215). */
int64_t orc_attn_block_backward(int64_t bs, int64_t heads, int64_t kv_heads, int64_t dim,
                                const double* q, const int64_t* qpos, const int64_t* qseg,
                                int64_t lq, const double* k, const double* v,
                                const int64_t* kpos, const int64_t* kseg, int64_t lk,
                                int causal, double scale, const double* out, const double* lse,
                                const double* dout, double* dq, double* dk, double* dv);
#endif
