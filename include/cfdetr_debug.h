/* cfdetr_debug.h — kernel-level entry points of libcfdetr.so for parity tests.
 *
 * These run ONE kernel of the hot path on caller buffers so tests can compare
 * intermediate layouts bit for bit (gather/select) and each tensor-core kernel
 * within tolerance, independently of the full call chain.  Same conventions as
 * cfdetr.h: device pointers unless h_-prefixed, bf16 as uint16_t, stream as void*,
 * enqueue-only, cfd_status results.  Not needed by normal users.
 */
#ifndef CFDETR_DEBUG_H_
#define CFDETR_DEBUG_H_

#include "cfdetr.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Epilogue selectors of cfdx_gemm (D = A . W^T, A [M,K] bf16, W [N,K] bf16 K-major):
 *   0  out_bf16[M,N] = bf16(D + bias)            (QKV projection)
 *   1  out_bf16[M,N] = bf16(GELU(D + bias))      (MLP1; GELU = z/2 (1 + erf(z/sqrt2)))
 *   2  out_f32[M,N] += D + bias                   (O-projection / MLP2 residual)
 * M is any positive count; N multiple of 64; K multiple of 64. */
cfd_status cfdx_gemm(int32_t M, int32_t N, int32_t K, const uint16_t *A, const uint16_t *W, const float *bias,
                     int32_t epi, uint16_t *out_bf16, float *out_f32, void *stream);

/* Residual + LayerNorm epilogue GEMM (EPI_F32_RESID_LN; N must be a single column tile,
 * N in {64, 128, 256}):  x[M,N] += A . W^T + bias;  ln_out[r] = bf16(LN(x[r]) * g + b) for
 * r < M and 0 for M <= r < ln_cap (pad rows).  staged = 1 selects the TMA-staged
 * epilogue (1 CTA/SM), 0 the direct-store one (2 CTAs/SM). */
cfd_status cfdx_gemm_resid_ln(int32_t M, int32_t N, int32_t K, const uint16_t *A, const uint16_t *W,
                              const float *bias, float *x, const float *ln_g, const float *ln_b, float eps,
                              uint16_t *ln_out, int32_t ln_cap, int32_t staged, void *stream);

/* Varlen multi-head attention over packed qkv [rows, 3d] (q | k | v) with
 * cu_seqlens [T+1]; writes O [rows, d] bf16 and, if lse != NULL, the natural-log
 * row log-sum-exp [nh, lse_ld].  rows_cap = rows allocated in qkv.  work_counter: a
 * caller-owned device int[2], zero before the first launch that uses it (each launch's last
 * CTA resets it), for dynamic item claiming; NULL = static round-robin.  One counter must not
 * be shared by launches that can run concurrently. */
cfd_status cfdx_attention(int32_t n_tasks, const int32_t *cu_seqlens, int32_t max_seqlen, int32_t rows_cap,
                          int32_t d_model, int32_t n_heads, const uint16_t *qkv, uint16_t *out, float *lse,
                          int32_t lse_ld, int32_t *work_counter, void *stream);

/* Row LayerNorm of fp32 x [M, d] -> bf16 y [M, d] (d in {64,128,256,512}). */
cfd_status cfdx_layernorm(int32_t M, int32_t d, const float *x, const float *g, const float *b, float eps,
                          uint16_t *y, void *stream);

/* Criticality score from packed equal-length frames: qkv [B*Nc, 3d], lse [nh, lse_ld]
 * -> scores [B, Nc]. */
cfd_status cfdx_score(int32_t n_frames, int32_t n_coarse, int32_t d_model, int32_t n_heads, const uint16_t *qkv,
                      int32_t rows_cap, const float *lse, int32_t lse_ld, float *scores, void *stream);

/* The B8 gather alone (ctx geometry): writes X coarse rows, cu_seqlens [T+1],
 * mixed_src, A_f [R, 3Pf^2] bf16, frow [R], fidx [R], meta [2] = {sum N_t, R}. */
cfd_status cfdx_gather(cfd_ctx *ctx, int32_t n_tasks, const uint16_t *images, const float *x0,
                       const int32_t *sel_idx, const int32_t *sel_count, float *X, int32_t *cu_seqlens,
                       int32_t *mixed_src, uint16_t *A_f, int32_t *frow, int32_t *fidx, int32_t *meta,
                       void *stream);

/* Launch probes.  Kernel classes: 0 attention, 1 score, 2 QKV GEMM, 3 O-proj GEMM,
 * 4 MLP1 GEMM, 5 MLP2 GEMM, 6 coarse-embed GEMM, 7 fine-embed GEMM, 8 layernorm,
 * 9 select, 10 gather, 11 im2col, 12 coarse meta.  After install, the i-th launch
 * (i < capacity) of class `kind` is bracketed by cudaEventRecordWithFlags(h_start[i] /
 * h_end[i], stream, cudaEventRecordExternal); the caller owns the (timing-enabled)
 * cudaEvent_t handles.  capacity 0 removes the probe.  cfdx_probe_count returns how
 * many launches were recorded since install. */
cfd_status cfdx_probe_install(int32_t kind, void *const *h_start, void *const *h_end, int32_t capacity);
int32_t cfdx_probe_count(int32_t kind);

/* Tuning switches for A/B measurement (every combination is parity-checked).  ctx != NULL:
 * the switch of that context only (each context starts at the defaults); ctx == NULL: the
 * switches the ctx-less debug entry points above use.
 *   key 0  attention kernel: 1 one query tile per CTA (v1; also used above 1024 tasks per launch),
 *          7 independent per-warpgroup items (task, head, 128-row tile), K/V rings, MMA and
 *          producer warps (v7, default)
 *   key 1  v7: how many of every 16 column pairs are exponentiated by the FMA-pipe
 *          polynomial instead of MUFU (0, 2 default, 4, 6, 8)
 *   key 2  fused MLP kernel on (1, default) / off (0)
 *   key 3  TMA-staged residual(+LayerNorm) epilogues on (1, default) / off (0)
 *   key 4  fused MLP (with the fused O-projection) as CTA pairs (cta_group::2, each SM holding half of
 *          every weight operand) on (1, default) / off (0); with key 11 = 0 the single-CTA kernel runs
 *   key 5  attention v7 warpgroup start stagger in cycles (700 default; values <= 0: none)
 *   key 7  weight-stationary QKV GEMM on (1, default) / off (0)
 *   key 11 O-projection + residual + LN2 fused into the MLP kernel on (1, default) / off (0)
 *   key 13 patch-embed GEMMs with one CTA per SM and a 4-stage ring (1, default) instead of
 *          two CTAs per SM with 2 stages (0)
 *   key 14 coarse patch embed gathering its A tiles straight from the image with a 5-D TMA
 *          tensor map (1, default; d = 256, 3Pc % 32 == 0) instead of im2col + GEMM (0)
 *   key 15 layer-0 LN1 of the coarse pass fused into the coarse embed epilogue (1, default)
 *          instead of a standalone LayerNorm launch (0)
 *   key 16 attention v7 dynamic item claiming through the call workspace's work counter (1,
 *          default) instead of the static round-robin (0)
 *   key 17 cap on the persistent kernels' grid size (0 = every SM, default)
 *   key 18 balanced persistent grids: the fewest CTAs with the same number of rounds (1) /
 *          min(units, SMs) (0, default)
 *   key 19 fused O-projection keeps x1 = x + o W_o + b_o in TMEM and the MLP's MMA2s
 *          accumulate onto it (1, default) / x1 stored and read back (0)
 *   key 21 attention v7: MMA-warp wait between barrier probes: 0, 8, 32 (default), 128 ns of
 *          sleep, 1 = try_wait (hardware suspend), 2 = busy test_wait loop
 *   key 24 attention v7: producer-warp sleep between barrier probes, ns (0..4096, default 256)
 *   key 22 attention v7: softmax warpgroups per CTA (3, or 4 default)
 *   key 23 QKV projection as CTA pairs (cta_group::2, half of each weight column block resident
 *          per SM, 8 A stages in flight) on (1, default) / off (0: one CTA per column block)
 *   key 25 image-sourced coarse patch embed as CTA pairs (cta_group::2, half of W_c per SM,
 *          12 stages) on (1, default) / off (0: one CTA per row block)
 * Other keys / values: CFD_E_ARG. */
cfd_status cfdx_set_option(cfd_ctx *ctx, int32_t key, int32_t value);

/* Number of kernels the library launched since load (host counter; for bench's
 * gpu_launches claim). */
int64_t cfdx_launch_count(void);

/* Pipeline event trace of the fused MLP kernel (debug library only, built with
 * -DCFD_TRACE): copies the SM clock64() stamps the last fused-MLP launch recorded for the
 * first two tiles of every CTA, 148 x 96 uint64 (layout in csrc/mlp_tc.cuh), into the host
 * buffer dst (n_words >= 148 * 96).  CFD_E_ARG when the library was built without tracing. */
cfd_status cfdx_mlp_trace(uint64_t* dst, int32_t n_words);
/* cfd_frames_from_u8 on a flat array of n elements (any n >= 0, including n % 16 != 0:
 * the ragged tail path); element i uses channel i mod 3. */
cfd_status cfdx_frames_u8(long long n, const uint8_t* src, const float* scale, const float* shift, uint16_t* dst,
                          void* stream);

/* Debug library only: copies the attention (v7) pipeline trace of the last launch
 * (ATTN_TRACE_WORDS = 148*4*2*12*8 + 148 uint64 clock64 values, layout in attn_common.cuh) to
 * host `dst`.  CFD_E_ARG in the release library or if n_words is too small. */
cfd_status cfdx_attn_trace(uint64_t* dst, int32_t n_words);

#ifdef __cplusplus
}
#endif
#endif /* CFDETR_DEBUG_H_ */
