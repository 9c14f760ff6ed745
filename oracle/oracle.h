/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference's
 * fused head-wise attention path, used as the CHECKER for the CUDA product
 * (never linked into it, never the thing measured). Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
 * oracle/liboracle.so.
 *
 * Parity pinning: every function here is checked against the reference
 * itself (oracle/_ref/libdfa2ref.so, compiled in place from
 * /root/reference/proj/src) and against golden vectors generated from it
 * (tests/golden/, tests/golden/gen_golden.py) in tests/test_oracle.py.
 *
 * Block masks are row-major uint8 [nb*nb], nb = ceil(n/B), as in
 * /root/reference/proj/include/dfa2/arrow.hpp:12-34.
 */
#ifndef DFA2_ORACLE_H
#define DFA2_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* build_arrow_mask, /root/reference/proj/src/arrow.cpp:113-153.
 * order: 0 visual_first, 1 text_first. Returns nb, or -1 on invalid input. */
int64_t orc_arrow_mask(int64_t nv, int64_t nt, int order, int64_t B, int64_t w,
                       uint8_t* active);
/* BlockMask::active_positions, arrow.cpp:95-104. */
int64_t orc_active_positions(const uint8_t* active, int64_t n, int64_t B);
/* plan_flops, dispatch.cpp:93-120. kinds: 0 full, 1 arrow, 2 cached. */
int64_t orc_plan_flops(int64_t H, int64_t d, int64_t nv, int64_t nt, int order,
                       int64_t B, const int32_t* kinds, const int64_t* windows);
/* streaming_block_pass over every query block, arrow.cpp:24-72 / 171-194,
 * scalar f32 (fixed-order dot/axpy). Returns 3 if a query block row is empty. */
int orc_sparse_forward_f32(const float* q, const float* k, const float* v, float* out,
                           int64_t n, int64_t d, const uint8_t* active, int64_t B);
/* attention_head_impl<double>, tensor.cpp:73-114: two-pass masked softmax
 * attention in f64 for the listed query rows (rows == NULL: all n rows).
 * active == NULL means unmasked. out is [nrows, d]. Returns 3 on a fully
 * masked row. */
int orc_attention_rows_f64(const float* q, const float* k, const float* v, int64_t n,
                           int64_t d, const uint8_t* active, int64_t B,
                           const int64_t* rows, int64_t nrows, double* out);
/* rse, calibrate.cpp:18-87 (mean -> sum_sq_dev -> numerator, sequential
 * double sums). mode 0 standard, 1 literal. Returns 5 on zero variance. */
int orc_rse_f32(const float* y_m, const float* y_o, int64_t numel, int mode, double* out);
/* Same on bf16 bit patterns (widened exactly to f32, then as above). */
int orc_rse_bf16(const uint16_t* y_m, const uint16_t* y_o, int64_t numel, int mode,
                 double* out);
/* f32 -> bf16 -> f32 round-to-nearest-even, in place (matches torch). */
void orc_round_bf16(float* x, int64_t numel);

#ifdef __cplusplus
}
#endif
#endif
