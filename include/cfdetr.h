/* cfdetr.h — C ABI of the B200 CF-DETR coarse-to-fine encoder hot path.
 *
 * The four calls follow the paper's statement of the problem (arXiv 2505.23317):
 *   cfd_coarse_encode   A1 coarse-to-fine inference, coarse stage: patch split +
 *                       embedding + encoder self-attention over the coarse tokens of
 *                       an image-level batch of frames (PAPER.md:78 §I A3, :119-122
 *                       §II-A, :220 §III-B A1); also emits the per-region
 *                       criticality score (reading R5) and the layer-0 token cache.
 *   cfd_select_regions  A2 region proposal as a per-region top-k or threshold
 *                       selection (§III-B A2; readings R5-R7).
 *   cfd_refine_encode   A2 selective fine split + coarse-token reuse + encoder re-run
 *                       on the mixed-resolution set of ONE task.
 *   cfd_batch_refine    A3 patch-level batch: the refine of T tasks with ragged token
 *                       counts in one launch per op, varlen/cu_seqlens instead of the
 *                       paper's zero padding (reading R11).
 *
 * Conventions
 *   - Every pointer is a DEVICE pointer unless its name starts with h_ (host).
 *   - `stream` is a cudaStream_t passed as void*; every call only enqueues work on
 *     it and returns (no host synchronisation inside any call, so calls can be
 *     captured in a CUDA graph).  A ctx is not thread-safe: one ctx per stream.
 *   - Tensors are dense row-major.  bf16 values are passed as uint16_t bit patterns.
 *   - Images are [.., H, W, 3] bf16 (HWC).  Patch vectors are ordered (py, px, ch)
 *     (reading R2).  Weight matrices are given (in, out) row-major.
 *   - The caller (e.g. torch) owns every tensor and the workspace; cfd_create copies
 *     and repacks the weights into ctx-owned device memory, so the caller may free
 *     its copies once the stream has synchronised after cfd_create.
 *   - Errors: host-detectable problems return a negative cfd_status before anything
 *     is enqueued; a CUDA launch failure returns CFD_E_CUDA; device-side input
 *     violations (sel_count > Nc, non-ascending or out-of-range sel_idx) set a device
 *     error word that cfd_check reports.  No C++ exception crosses the ABI.
 *   - Numerics: bf16 GEMM operands (RNE), fp32 accumulation, fp32 residual stream,
 *     LN statistics and softmax state, bf16 P into the PV product; fp32 outputs
 *     (reading R13).
 */
#ifndef CFDETR_H_
#define CFDETR_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  CFD_OK = 0,
  CFD_E_ARG = -1,         /* null pointer, non-positive count, k > Nc, bad mode */
  CFD_E_SHAPE = -2,       /* H or W not a multiple of Pc, Pc not a multiple of Pf, d % nh */
  CFD_E_UNSUPPORTED = -3, /* dh != 32, d not in {64,128,256,512}, Nc > 4096, ... */
  CFD_E_CAPACITY = -4,    /* n_tasks > max_tasks, or workspace too small */
  CFD_E_CUDA = -5,        /* a CUDA API call or kernel launch failed */
  CFD_E_DEVICE = -6       /* a kernel flagged invalid device-side input (cfd_check) */
} cfd_status;

/* Model geometry.  score_layer in [0, n_layers): the layer whose attention map
 * scores the regions (default n_layers-1).  max_tasks bounds n_frames / n_tasks. */
typedef struct {
  int32_t img_h, img_w;
  int32_t patch_coarse; /* Pc */
  int32_t patch_fine;   /* Pf, Pc % Pf == 0, m = Pc/Pf */
  int32_t d_model;      /* d */
  int32_t n_heads;      /* nh, dh = d/nh must be 32 */
  int32_t n_layers;     /* L */
  int32_t d_ff;         /* F (multiple of 64) */
  int32_t score_layer;
  int32_t max_tasks;
  float ln_eps;         /* 1e-6 */
} cfd_config;

/* One pre-LN encoder block (reading R4); matrices bf16 (in, out), vectors fp32. */
typedef struct {
  const uint16_t *w_qkv; /* [d, 3d]  columns: q | k | v, head h at [h*dh, (h+1)*dh) */
  const uint16_t *w_o;   /* [d, d] */
  const uint16_t *w_1;   /* [d, F] */
  const uint16_t *w_2;   /* [F, d] */
  const float *b_qkv, *b_o, *b_1, *b_2;          /* [3d], [d], [F], [d] */
  const float *ln1_g, *ln1_b, *ln2_g, *ln2_b;    /* [d] each */
} cfd_layer_weights;

typedef struct {
  const uint16_t *w_embed_c; /* [3Pc^2, d] coarse patch embedding (reading R1) */
  const uint16_t *w_embed_f; /* [3Pf^2, d] fine patch embedding */
  const float *b_embed_c;    /* [d] */
  const float *b_embed_f;    /* [d] */
  const float *pe_c;         /* [Nc, d] fixed positional table, coarse raster (reading R3) */
  const float *pe_f;         /* [Nf, d] fine raster */
  const cfd_layer_weights *h_layers; /* HOST array [n_layers] of device pointers */
} cfd_weights;

typedef enum { CFD_SELECT_TOPK = 0, CFD_SELECT_THRESHOLD = 1 } cfd_select_mode;

typedef struct cfd_ctx cfd_ctx;

/* Validate cfg, allocate ctx-owned device memory, repack weights (enqueued on stream). */
cfd_status cfd_create(const cfd_config *cfg, const cfd_weights *w, void *stream, cfd_ctx **out);
/* Free ctx memory (synchronises the device). NULL is a no-op. */
cfd_status cfd_destroy(cfd_ctx *ctx);

/* Geometry and the workspace a call with n_tasks frames/tasks needs:
 *   *h_Nc = (H/Pc)(W/Pc), *h_Nf = m^2 Nc, *h_max_tokens = n_tasks * Nf (capacity of
 *   packed refine outputs), *h_workspace_bytes = bytes for ws.  Any output may be NULL. */
cfd_status cfd_query(const cfd_ctx *ctx, int32_t n_tasks, int32_t *h_Nc, int32_t *h_Nf, int32_t *h_max_tokens,
                     size_t *h_workspace_bytes);

/* A1 coarse pass over n_frames equal-size frames (image-level batch).
 *   images    [B, H, W, 3] bf16
 *   x0        [B, Nc, d] fp32 out: layer-0 coarse tokens (patch.W_c + b_c + PE_c), the
 *             cache refine reuses for unselected regions (reading R8)
 *   y         [B, Nc, d] fp32 out: encoder output
 *   scores    [B, Nc] fp32 out or NULL: criticality score at cfg.score_layer
 *   layer_out [L, B, Nc, d] fp32 out or NULL: residual stream after every layer
 *   ws        workspace of >= cfd_query(n_frames) bytes (256-byte aligned) */
cfd_status cfd_coarse_encode(cfd_ctx *ctx, int32_t n_frames, const uint16_t *images, float *x0, float *y,
                             float *scores, float *layer_out, void *ws, size_t ws_bytes, void *stream);

/* A2 selection over n_tasks score rows.
 *   scores    [T, Nc] fp32
 *   TOPK:      h_k [T] host ints, 0 <= k_t <= Nc; ties -> lower index; NaN lowest; -0 == +0
 *   THRESHOLD: regions with score > threshold (strict)
 *   sel_idx   [T, Nc] int32 out: selected region indices ascending in the first
 *             sel_count[t] entries, -1 after;  sel_count [T] int32 out. */
cfd_status cfd_select_regions(cfd_ctx *ctx, int32_t n_tasks, const float *scores, cfd_select_mode mode,
                              const int32_t *h_k, float threshold, int32_t *sel_idx, int32_t *sel_count,
                              void *stream);

/* A2/A3 patch-level refine of n_tasks tasks, packed varlen.
 *   images    [T, H, W, 3] bf16;  x0 [T, Nc, d] (from cfd_coarse_encode)
 *   sel_idx/sel_count as produced by cfd_select_regions
 *   h_token_counts [T] host hint of N_t = Nc + (m^2-1) k_t, or NULL (capacity launch)
 *   y         [cap, d] fp32 out, cap = T*Nf: task t occupies rows [cu[t], cu[t+1])
 *   cu_seqlens[T+1] int32 out;  mixed_src [cap] int32 out: >= 0 coarse index, < 0 is
 *             -1 - fine index (reading R10)
 *   layer_out [L, cap, d] or NULL.  Tasks never attend to each other; the result of
 *   each task equals its cfd_refine_encode result bit for bit. */
cfd_status cfd_batch_refine(cfd_ctx *ctx, int32_t n_tasks, const uint16_t *images, const float *x0,
                            const int32_t *sel_idx, const int32_t *sel_count, const int32_t *h_token_counts,
                            float *y, int32_t *cu_seqlens, int32_t *mixed_src, float *layer_out, void *ws,
                            size_t ws_bytes, void *stream);

/* NEXT row f4 — the paper's pad-to-max patch-level batch (§III-B A3 "padding
 * is applied to equalize them"; :466 [draft]), the baseline the varlen cfd_batch_refine is
 * measured against.  Every task occupies max_tokens rows: rows [t*max_tokens, t*max_tokens +
 * N_t) hold its mixed tokens (the same order as cfd_batch_refine), the remaining rows are zero
 * pad tokens; every layer runs over all T*max_tokens rows, and attention covers all
 * max_tokens keys of the task with the pad keys masked (exp -> 0; reading R11: unmasked pad
 * keys would receive softmax weight).  Per task, rows [0, N_t) equal cfd_batch_refine's output
 * bit for bit.
 *   max_tokens  >= every N_t = Nc + (m^2-1) k_t and <= Nf (host value; a task with N_t >
 *             max_tokens sets the device error word, see cfd_check)
 *   y         [T*max_tokens, d] fp32 out;  cu_seqlens [T+1] out = t*max_tokens;
 *   kv_len    [T] int32 out = N_t;  mixed_src [T*max_tokens] out (pad rows INT32_MIN)
 *   layer_out [L, T*max_tokens, d] or NULL;  workspace: cfd_query(ctx, n_tasks).
 * Errors as cfd_batch_refine; CFD_E_ARG if max_tokens is outside [Nc, Nf]. */
cfd_status cfd_batch_refine_padded(cfd_ctx *ctx, int32_t n_tasks, const uint16_t *images, const float *x0,
                                   const int32_t *sel_idx, const int32_t *sel_count, int32_t max_tokens, float *y,
                                   int32_t *cu_seqlens, int32_t *kv_len, int32_t *mixed_src, float *layer_out,
                                   void *ws, size_t ws_bytes, void *stream);

/* cfd_batch_refine with T = 1 (y capacity Nf rows, cu_seqlens [2]). */
cfd_status cfd_refine_encode(cfd_ctx *ctx, const uint16_t *image, const float *x0, const int32_t *sel_idx,
                             const int32_t *sel_count, float *y, int32_t *mixed_src, int32_t *cu_seqlens,
                             float *layer_out, void *ws, size_t ws_bytes, void *stream);

/* NEXT row f2 — A1 hardness gate: for each frame, queries with confidence
 * c > c_hi (0.8: large, safety-critical objects) are excluded and the remaining
 * confidences averaged; the frame is easy (hard[b] = 0: coarse result suffices, refine
 * with k = 0) if that mean is below tau_easy (0.05), else hard (1).  No remaining query ->
 * easy.  conf [B, Q] fp32; hard [B] int32 out.  The mean is evaluated as an fp64
 * sequential sum in query order compared with tau_easy * n (bit-exact decision). */
cfd_status cfd_hardness(cfd_ctx *ctx, int32_t n_frames, int32_t n_queries, const float *conf, float c_hi,
                        float tau_easy, int32_t *hard, void *stream);

/* NEXT row f1 — box-driven region proposal: ROIs from the boxes of
 * intermediate-confidence queries (c_lo < c <= c_hi; 0.05 / 0.8).
 * boxes [B, Q, 4] fp32 (cx, cy, w, h) normalised to the image; conf [B, Q] fp32;
 * scores [B, Nc] fp32 out = number of (query, pixel) pairs inside each coarse cell (an
 * exact integer).  cfd_select_regions(THRESHOLD, 0) then selects every cell an
 * intermediate box touches; TOPK ranks them by coverage.  n_queries <= 4096. */
cfd_status cfd_box_scores(cfd_ctx *ctx, int32_t n_frames, int32_t n_queries, const float *boxes, const float *conf,
                          float c_lo, float c_hi, float *scores, void *stream);

/* NEXT row f3 — DETR decoder cross-attention + detection heads ("each
 * query attends to the encoded patch features (through encoder-decoder cross-attention) ...
 * and each query outputs a bounding box with a class label ... and a confidence score";
 * 128 object queries).  One block, reading R24:
 *   h_q = LN_q(Q0);  q = h_q W_q + b_q                       (Q0: n_queries learned queries)
 *   per task t:  h_m = LN_m(y_t);  [k | v] = h_m W_kv + b_kv  (y_t: task t's encoder output)
 *   o = concat_h softmax(q_h k_h^T / sqrt(dh)) v_h;  z = Q0 + o W_o + b_o
 *   [box | c] = sigmoid(z W_head + b_head)                   (box = (cx, cy, w, h), c = confidence)
 * Weights (device pointers, copied into the ctx by cfd_set_decoder, caller may free them
 * after the stream syncs): queries fp32 [Q, d]; ln_q / ln_m gamma, beta fp32 [d]; w_q bf16
 * [d, d], w_kv bf16 [d, 2d], w_o bf16 [d, d], w_head fp32 [d, 5], all (in, out); biases fp32.
 * Q <= 128.  Errors: CFD_E_ARG (null / Q out of range), CFD_E_UNSUPPORTED (dh != 32). */
typedef struct {
  int32_t n_queries;
  const float *queries;
  const float *ln_q_g, *ln_q_b, *ln_m_g, *ln_m_b;
  const uint16_t *w_q, *w_kv, *w_o;
  const float *b_q, *b_kv, *b_o;
  const float *w_head, *b_head;
} cfd_decoder_weights;
cfd_status cfd_set_decoder(cfd_ctx *ctx, const cfd_decoder_weights *w, void *stream);

/* Decode n_tasks packed encoder outputs (the y / cu_seqlens of cfd_coarse_encode (cu =
 * [0, Nc, 2Nc, ...]) or cfd_batch_refine).  y fp32 [rows, d] device; cu_seqlens int32
 * [T+1] device; h_max_tokens: host upper bound of cu_seqlens[T] (sizes the launches).
 * Out (device): z fp32 [T, Q, d] (decoded query embeddings, may be NULL), boxes fp32
 * [T, Q, 4], conf fp32 [T, Q].  ws / ws_bytes: a workspace from cfd_query for >= n_tasks
 * tasks.  CFD_E_ARG without cfd_set_decoder. */
cfd_status cfd_decode(cfd_ctx *ctx, int32_t n_tasks, const float *y, const int32_t *cu_seqlens, int32_t h_max_tokens,
                      float *z, float *boxes, float *conf, void *ws, size_t ws_bytes, void *stream);

/* Frame ingest (serving path; not a step of the paper's method, which starts from camera
 * images, "images ... from the cameras"): 8-bit HWC frames -> the bf16 HWC
 * frames cfd_coarse_encode / cfd_batch_refine read, so a host uploads 1 byte per channel
 * value instead of 2.  Element i (channel c = i mod 3) of each frame:
 *   images[i] = bf16_rn( fp32_fma(src[i], scale[c], shift[c]) )
 * i.e. one fp32 fused multiply-add (single rounding) then round-to-nearest-even to bf16; with
 * scale = 1 / (255 std_c) and shift = -mean_c / std_c this is the usual (p/255 - mean)/std.
 * src uint8 [n_frames, H, W, 3] device; images uint16 (bf16 bits) [n_frames, H, W, 3]
 * device (may be the buffer later passed to the encode calls); scale, shift: HOST arrays of
 * 3 floats, read during the call (capture-safe: the values are baked into the launch).
 * n_frames = 0 is a no-op.  Errors: CFD_E_ARG (null pointer, n_frames < 0). */
cfd_status cfd_frames_from_u8(cfd_ctx *ctx, int32_t n_frames, const uint8_t *src, const float *scale,
                              const float *shift, uint16_t *images, void *stream);

/* Synchronise `stream`; return CFD_E_DEVICE (and clear the word) if a kernel flagged
 * invalid device-side input since the last check, CFD_E_CUDA on a sticky CUDA error. */
cfd_status cfd_check(cfd_ctx *ctx, void *stream);

const char *cfd_status_str(cfd_status s);

/* Library build identification string (static storage). */
const char *cfd_version(void);

#ifdef __cplusplus
}
#endif
#endif /* CFDETR_H_ */
