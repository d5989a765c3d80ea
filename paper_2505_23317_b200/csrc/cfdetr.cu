// cfdetr.cu — host side of libcfdetr.so: the C ABI of include/cfdetr.h and
// include/cfdetr_debug.h.  Owns weight repacking, TMA descriptors, workspace
// carving and the launch sequence of every call:
//
//   cfd_coarse_encode : im2col -> B1 embed GEMM -> L x [LN1 -> QKV GEMM -> attention
//                       (-> score at score_layer) -> O GEMM(+res) -> LN2 -> MLP1(GELU)
//                       -> MLP2(+res)]
//   cfd_select_regions: B7 select
//   cfd_batch_refine  : B8 gather -> B9 fine embed GEMM (row scatter) -> L x [same
//                       block, varlen attention over cu_seqlens]
// All launches go to the caller's stream; no host synchronisation.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <set>
#include <utility>
#include <vector>

#include "../../include/cfdetr.h"
#include "../../include/cfdetr_debug.h"
#include "attn_tc.cuh"
#include "attn_common.cuh"
#include "attn7_tc.cuh"
#include "gemm_tc.cuh"
#include "misc_kernels.cuh"
#include "mlp_tc.cuh"
#include "score_tc.cuh"

using namespace cfd;

namespace {

std::atomic<int64_t> g_launches{0};

// ---------------------------------------------------------------- launch probes
// Optional per-kernel-class CUDA event pairs (cfdx_probe_install): every launch of a
// probed class is bracketed by cudaEventRecordWithFlags(..., External) on the
// launching stream, so bench.py can time the dominant kernel live.
constexpr int kProbeKinds = 16;
struct Probe {
  std::vector<cudaEvent_t> start, end;
  int count = 0;
};
Probe g_probe[kProbeKinds];

// cudaEventRecordExternal is only valid while the stream is capturing a graph.
inline void probe_record(cudaEvent_t e, cudaStream_t s) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &cs);
  if (cs == cudaStreamCaptureStatusActive) cudaEventRecordWithFlags(e, s, cudaEventRecordExternal);
  else cudaEventRecord(e, s);
}
inline void probe_begin(int kind, cudaStream_t s) {
  if (kind < 0 || kind >= kProbeKinds) return;
  Probe& p = g_probe[kind];
  if (p.count < (int)p.start.size()) probe_record(p.start[p.count], s);
}
inline void probe_end(int kind, cudaStream_t s) {
  if (kind < 0 || kind >= kProbeKinds) return;
  Probe& p = g_probe[kind];
  if (p.count < (int)p.end.size()) probe_record(p.end[p.count++], s);
}

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                     const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                     CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

PFN_encodeTiled get_encode_fn() {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  }
  return fn;
}

// 2-D bf16 tensor map: inner dim `inner` elements (contiguous), `outer` rows with
// row stride `ld` elements, box {box_inner, box_outer}.
bool make_tmap(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint64_t ld, uint32_t box_inner,
               uint32_t box_outer, CUtensorMapSwizzle sw, bool fp32 = false) {
  PFN_encodeTiled enc = get_encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld * (fp32 ? 4 : 2)};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, fp32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                   const_cast<void*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// Tuning switches (cfdx_set_option, include/cfdetr_debug.h).  Every context carries its own
// copy (set per ctx); the ctx-less debug entry points use g_dbg_opts.  Defaults = the measured
// best configuration.
struct Opts {
  int attn_variant = 7;   // 1: one q-tile per CTA (v1; also the fallback above ATTN7_MAX_T tasks),
                          // 7: independent per-warpgroup items and pipelines (v7, default)
  int attn_npp = 2;       // v4 / v7: polynomial-exp pairs of every 16 (v7: 2 measured best)
  int attn_stagger = 700; // v4 / v7: warpgroup start stagger in cycles (v7: 700 measured best:
                          // 58.2 vs 60.5 us at 700 x 32); -1 / -2 trace modes (debug library)
  int attn_dyn = 1;       // v4: dynamic item claiming through the workspace work counter (16)
  int fused_mlp = 1;      // fused MLP kernel (d == 256) instead of two GEMM launches (2)
  int staged_epi = 1;     // TMA-staged residual + LayerNorm epilogues (3)
  int mlp_cluster = 1;    // fused MLP (+ fused O-projection) as CTA pairs (cta_group::2) (4; 52.3 -> 49.2 us)
  int gemm_bres = 1;      // weight-stationary QKV GEMM (7)
  int fuse_oproj = 1;     // O-projection + residual + LN2 inside the fused MLP kernel (11)
  int embed_mode0 = 1;    // patch-embed GEMMs: 1 CTA/SM, 4-stage ring (13)
  int embed_img = 1;      // coarse patch embed gathers A from the image by TMA, no im2col (14)
  int embed_ln = 1;       // layer-0 LN1 fused into the coarse embed epilogue (15)
  int sm_cap = 0;         // cap on the persistent grids (0 = all SMs) (17)
  int balanced_grid = 0;  // fewest CTAs with the same number of rounds (18)
  int keep_x1 = 1;        // fused O-projection: x1 stays in TMEM, MMA2 accumulates onto it (19)
  int attn_sleep = 32;    // v7: MMA / producer warp sleep when idle, ns (21: 0, 32, 128)
  int attn_psleep = 256;  // v7: the producer warp's sleep between barrier probes, ns (24: 0..4096)
  int attn_nwg = 4;       // v7: softmax warpgroups per CTA (22: 3 or 4)
  int qkv_pair = 1;       // QKV projection as CTA pairs, half of the weights resident per SM (23)
  int embed_pair = 1;     // image-sourced coarse patch embed as CTA pairs, half of W_c per SM (25)
};
Opts g_dbg_opts;

int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev;
}

// SM count of the current device (cached per device)
int device_sms() {
  static std::atomic<int> cache[64];
  const int dev = current_device();
  if (dev < 0 || dev >= 64) return 148;
  int n = cache[dev].load();
  if (!n) {
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
    cache[dev].store(n);
  }
  return n;
}
int num_sms(const Opts& o) {
  const int n = device_sms();
  return o.sm_cap > 0 ? std::min(o.sm_cap, n) : n;
}

// cudaFuncAttributeMaxDynamicSharedMemorySize is a per-device property of a kernel: set it
// once per (kernel, device).
template <typename K>
cudaError_t ensure_smem_attr(K* kern, int smem) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  const std::pair<const void*, int> key{reinterpret_cast<const void*>(kern), current_device()};
  std::lock_guard<std::mutex> lk(mu);
  if (done.count(key)) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e == cudaSuccess) done.insert(key);
  return e;
}

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Persistent grid for `units` equal work units on at most `slots` CTAs: the fewest CTAs that
// keep the same number of rounds (ceil(units / slots)), so a launch whose last round would
// be partial leaves whole SMs to a concurrent stream instead of idling them in its tail
// (option 18; e.g. 256 attention items: 128 CTAs x 2 rounds instead of 148 CTAs with 40 idle
// in round 2).
// off by default: 2-stream step 1.385 vs 1.389 ms (noise), 1-stream 1.479 vs 1.462 ms
inline int balanced_grid(const Opts& o, int units, int slots) {
  if (units <= 0) return 1;
  if (!o.balanced_grid || units <= slots) return std::min(units, slots);
  const int rounds = (units + slots - 1) / slots;
  return (units + rounds - 1) / rounds;
}

// ------------------------------------------------------------------ launches
template <typename... KArgs, typename... Args>
cudaError_t launch_ex(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
  kern<<<grid, block, smem, s>>>(std::forward<Args>(args)...);
  return cudaGetLastError();
}


// ------------------------------------------------------------------ GEMM dispatch
template <int BN>
constexpr int gemm_stages() { return BN == 256 ? 4 : BN == 128 ? 6 : 8; }
template <int BN>  // with the 32 KB bf16 output staging area
constexpr int gemm_stages_stg() { return BN == 256 ? 3 : BN == 128 ? 5 : 7; }

// mode 0: 1 CTA/SM, 8 epilogue warps, double-buffered accumulator (many tiles);
//         for EPI_F32_RESID_LN a 2-stage ring and the TMA-staged residual epilogue
// mode 1: 2 CTAs/SM, 4 epilogue warps, single accumulator, 2-stage ring (N = d GEMMs)
// mode 2 (BRES): mode 0 with the CTA's [BN, 256] weight slice resident in shared memory
//         (bf16 outputs, K = 256): each CTA keeps one column block and walks row blocks, so
//         the per-SM operand stream is A only (64 KB per 128x256 tile instead of 192 KB)
// mode 3 (IMG): mode 0 for the coarse patch embed with A gathered from the image by a 5-D
//         tensor map (no im2col), 32-wide k-blocks, 8-stage ring of 8 + 16 KB
template <int BN, int EPI, int MODE>
cudaError_t launch_gemm_t(const Opts& o, const CUtensorMap& ta, const CUtensorMap& tb, const GemmParams& p,
                          int rows_for_grid, cudaStream_t s, const CUtensorMap* tx, const CUtensorMap* tln) {
  constexpr bool kImg = MODE == 3;
  constexpr bool kBres = MODE == 2;
  constexpr bool kTmaEpi = (EPI == EPI_F32_RESID_LN && MODE != 1);
  constexpr bool kStgOut = (EPI == EPI_BF16_BIAS || EPI == EPI_BF16_BIAS_GELU) && MODE != 1;
  constexpr int EW = MODE == 1 ? 4 : 8;
  constexpr int NACC = MODE == 1 ? 1 : 2;
  // BRES: 4 A stages (64 KB in flight: the A tiles come from L2 / DRAM at ~1-2 us latency)
  // with one 2 KB output staging buffer per epilogue warp
  constexpr int ST = kImg ? 8 : kBres ? 4 : (MODE == 1 || kTmaEpi) ? 2 : kStgOut ? gemm_stages_stg<BN>() : gemm_stages<BN>();
  auto kern = gemm_tc_kernel<BN, ST, EPI, EW, NACC, kBres, kImg>;
  using SM = GemmSmem<BN, ST, NACC, kBres, kImg ? 32 : GEMM_BK>;
  constexpr int smem = kTmaEpi ? SM::TOTAL_TMA_EPI : (kStgOut && kBres) ? SM::TOTAL_STG_OUT1
                       : kStgOut ? SM::TOTAL_STG_OUT : SM::TOTAL;
  static_assert(smem <= 232448, "shared memory budget");
  CUtensorMap tout;
  if constexpr (kStgOut) {  // bf16 output [m_cap, N], 32 x 32 boxes
    if (!make_tmap(&tout, p.out_bf16, p.N, p.m_cap, p.N, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B))
      return cudaErrorInvalidValue;
    tx = &tout;
  }
  if (cudaError_t e = ensure_smem_attr(kern, smem); e != cudaSuccess) return e;
  const int rpt = kImg ? p.img_rb * p.img_gw : GEMM_BM;
  const int tiles = ((rows_for_grid + rpt - 1) / rpt) * (p.N / BN);
  const int slots = num_sms(o) * (MODE == 1 ? 2 : 1);
  int grid = balanced_grid(o, tiles, slots);
  if constexpr (kBres) {  // whole column-block groups, each balanced over its row blocks
    const int nt = p.N / BN, mt = (rows_for_grid + rpt - 1) / rpt;
    grid = balanced_grid(o, mt, std::max(1, slots / nt)) * nt;
  }
  cudaError_t le = launch_ex(kern, dim3(grid), dim3(64 + 32 * EW), smem, s, ta, tb, p, tx ? *tx : ta, tln ? *tln : ta);
  ++g_launches;
  return le != cudaSuccess ? le : cudaGetLastError();
}

// Image-sourced coarse patch embed as CTA pairs (gemm_tc_kernel IMG + PAIR): each CTA gathers its
// own row block of patches and half of every W_c k-block (128 of the 256 columns), the leader issues
// M = 256 cta_group::2 MMAs, each CTA's epilogue finishes its own rows (PE, x0, layer-0 LN1):
// per-SM weight ingress halves (W_c is 1.5 MB per row block).
cudaError_t launch_embed_pair(const Opts& o, const CUtensorMap& ta, const CUtensorMap& tb_half, const GemmParams& p,
                              int rows_for_grid, cudaStream_t s) {
  constexpr int ST = 8;  // 8 / 12 / 6 stages: 135.7 / 139.0 / 139.9 us per 128 frames
  auto kern = gemm_tc_kernel<256, ST, EPI_EMBED_COARSE, 8, 2, false, true, true>;
  using SM = GemmSmem<256, ST, 2, false, 32, true>;
  constexpr int smem = SM::TOTAL;
  static_assert(smem <= 232448, "shared memory budget");
  if (cudaError_t e = ensure_smem_attr(kern, smem); e != cudaSuccess) return e;
  const int rpt = p.img_rb * p.img_gw;
  const int units = ((rows_for_grid + rpt - 1) / rpt + 1) / 2;  // row-block pairs
  const int pairs = balanced_grid(o, units, std::max(1, num_sms(o) / 2));
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(2 * pairs);
  lc.blockDim = dim3(64 + 32 * 8);
  lc.dynamicSmemBytes = smem;
  lc.stream = s;
  cudaLaunchAttribute la[1];
  la[0].id = cudaLaunchAttributeClusterDimension;
  la[0].val.clusterDim.x = 2;
  la[0].val.clusterDim.y = 1;
  la[0].val.clusterDim.z = 1;
  lc.attrs = la;
  lc.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&lc, kern, ta, tb_half, p, ta, ta);
  ++g_launches;
  return e != cudaSuccess ? e : cudaGetLastError();
}

// QKV projection as CTA pairs (gemm_tc_kernel PAIR): bf16 out + bias, K = 256, N = 3d with
// BN = 256 column blocks; 2-CTA clusters, (74 / n_tiles) * n_tiles clusters at most.
cudaError_t launch_qkv_pair(const Opts& o, const CUtensorMap& ta, const CUtensorMap& tb_half, const GemmParams& p,
                            int rows_for_grid, cudaStream_t s) {
  constexpr int ST = 8;
  auto kern = gemm_tc_kernel<256, ST, EPI_BF16_BIAS, 8, 2, true, false, true>;
  using SM = GemmSmem<256, ST, 2, true, GEMM_BK, true>;
  constexpr int smem = SM::TOTAL_STG_OUT1;
  static_assert(smem <= 232448, "shared memory budget");
  if (cudaError_t e = ensure_smem_attr(kern, smem); e != cudaSuccess) return e;
  CUtensorMap tout;  // bf16 output [m_cap, N], 32 x 32 boxes
  if (!make_tmap(&tout, p.out_bf16, p.N, p.m_cap, p.N, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B)) return cudaErrorInvalidValue;
  const int nt = p.N / 256, mt = (rows_for_grid + GEMM_BM - 1) / GEMM_BM;
  const int pairs_per_col = std::max(1, std::min((mt + 1) / 2, (num_sms(o) / 2) / nt));
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(2 * pairs_per_col * nt);
  lc.blockDim = dim3(64 + 32 * 8);
  lc.dynamicSmemBytes = smem;
  lc.stream = s;
  cudaLaunchAttribute la[1];
  la[0].id = cudaLaunchAttributeClusterDimension;
  la[0].val.clusterDim.x = 2;
  la[0].val.clusterDim.y = 1;
  la[0].val.clusterDim.z = 1;
  lc.attrs = la;
  lc.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&lc, kern, ta, tb_half, p, tout, ta);
  ++g_launches;
  return e != cudaSuccess ? e : cudaGetLastError();
}

template <int EPI>
cudaError_t launch_gemm_bn(const Opts& o, int BN, const CUtensorMap& ta, const CUtensorMap& tb, const GemmParams& p,
                           int rows, cudaStream_t s, const CUtensorMap* tx, const CUtensorMap* tln) {
  // N = BN: a single column tile per row block -> the 2-CTA/SM configuration, except the
  // residual+LN epilogue with staging maps, which runs 1 CTA/SM with TMA-staged I/O
  // the patch embeds (K = 3Pc^2 / 3Pf^2, long k loops over ~100 tiles) keep one CTA per SM with a
  // 4-stage ring when embed_mode0 (option 13): the k loop is latency-bound with 2 stages
  const bool embed = (EPI == EPI_EMBED_COARSE || EPI == EPI_EMBED_FINE) && o.embed_mode0;
  if (p.N == BN && !(EPI == EPI_F32_RESID_LN && tx && tln) && !embed) {
    switch (BN) {
      case 256: return launch_gemm_t<256, EPI, 1>(o, ta, tb, p, rows, s, tx, tln);
      case 128: return launch_gemm_t<128, EPI, 1>(o, ta, tb, p, rows, s, tx, tln);
      default: return launch_gemm_t<64, EPI, 1>(o, ta, tb, p, rows, s, tx, tln);
    }
  }
  if constexpr (EPI == EPI_BF16_BIAS) {
    if (o.gemm_bres && BN == 256 && p.K == GEMM_BRES_KB * GEMM_BK)
      return launch_gemm_t<256, EPI, 2>(o, ta, tb, p, rows, s, tx, tln);
  }
  switch (BN) {
    case 256: return launch_gemm_t<256, EPI, 0>(o, ta, tb, p, rows, s, tx, tln);
    case 128: return launch_gemm_t<128, EPI, 0>(o, ta, tb, p, rows, s, tx, tln);
    default: return launch_gemm_t<64, EPI, 0>(o, ta, tb, p, rows, s, tx, tln);
  }
}

int pick_bn(int N) { return (N % 256 == 0) ? 256 : (N % 128 == 0) ? 128 : 64; }

cudaError_t launch_gemm_impl(const Opts& o, int epi, const CUtensorMap& ta, const CUtensorMap& tb,
                             const GemmParams& p, int rows, cudaStream_t s, const CUtensorMap* tx,
                             const CUtensorMap* tln) {
  const int BN = pick_bn(p.N);
  switch (epi) {
    case EPI_BF16_BIAS: return launch_gemm_bn<EPI_BF16_BIAS>(o, BN, ta, tb, p, rows, s, nullptr, nullptr);
    case EPI_BF16_BIAS_GELU: return launch_gemm_bn<EPI_BF16_BIAS_GELU>(o, BN, ta, tb, p, rows, s, nullptr, nullptr);
    case EPI_F32_RESID: return launch_gemm_bn<EPI_F32_RESID>(o, BN, ta, tb, p, rows, s, nullptr, nullptr);
    case EPI_EMBED_COARSE: return launch_gemm_bn<EPI_EMBED_COARSE>(o, BN, ta, tb, p, rows, s, nullptr, nullptr);
    case EPI_F32_RESID_LN: return launch_gemm_bn<EPI_F32_RESID_LN>(o, BN, ta, tb, p, rows, s, tx, tln);
    default: return launch_gemm_bn<EPI_EMBED_FINE>(o, BN, ta, tb, p, rows, s, nullptr, nullptr);
  }
}

// probe kinds (cfdetr_debug.h)
enum : int { PK_ATTN = 0, PK_SCORE = 1, PK_QKV = 2, PK_OPROJ = 3, PK_MLP1 = 4, PK_MLP2 = 5, PK_EMBED_C = 6,
             PK_EMBED_F = 7, PK_LN = 8, PK_SELECT = 9, PK_GATHER = 10, PK_IM2COL = 11, PK_META = 12 };

cudaError_t launch_gemm(const Opts& o, int epi, const CUtensorMap& ta, const CUtensorMap& tb, const GemmParams& p,
                        int rows, cudaStream_t s, int kind = -1, const CUtensorMap* tx = nullptr,
                        const CUtensorMap* tln = nullptr) {
  probe_begin(kind, s);
  cudaError_t e = launch_gemm_impl(o, epi, ta, tb, p, rows, s, tx, tln);
  probe_end(kind, s);
  return e;
}

// B tensor map for a K-major weight [N, K]
// 5-D map over HWC bf16 frames [B][H][W][3] for the image-sourced coarse embed:
//   d0 = 32 elements of a pixel segment, d1 = segment third j (3Pc/32), d2 = patch column cx,
//   d3 = pixel row in the patch py, d4 = coarse row R = b * gh + cy;  box {32, 1, gw, 1, rb}
//   -> rb * gw rows of 64 B, row (R, cx) = A[patch][(py*Pc + px)*3 + ch] for the 32 k of (py, j)
bool make_img_map(CUtensorMap* m, const void* img, int B, int H, int W, int Pc, int rb) {
  PFN_encodeTiled enc = get_encode_fn();
  if (!enc) return false;
  const int gw = W / Pc, gh = H / Pc, thirds = 3 * Pc / 32;
  cuuint64_t dims[5] = {32, (cuuint64_t)thirds, (cuuint64_t)gw, (cuuint64_t)Pc, (cuuint64_t)B * gh};
  cuuint64_t strides[4] = {64, (cuuint64_t)3 * Pc * 2, (cuuint64_t)W * 3 * 2, (cuuint64_t)Pc * W * 3 * 2};
  cuuint32_t box[5] = {32, 1, (cuuint32_t)gw, 1, (cuuint32_t)rb};
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(img), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool make_wmap(CUtensorMap* m, const void* w, int N, int K) {
  return make_tmap(m, w, K, N, K, GEMM_BK, pick_bn(N), CU_TENSOR_MAP_SWIZZLE_128B);
}
bool make_amap(CUtensorMap* m, const void* a, int rows, int K) {
  return make_tmap(m, a, K, rows, K, GEMM_BK, GEMM_BM, CU_TENSOR_MAP_SWIZZLE_128B);
}
bool make_qkvmap(CUtensorMap* m, const void* qkv, int rows, int d, int box_rows = 128) {
  return make_tmap(m, qkv, 3 * d, rows, 3 * d, 32, box_rows, CU_TENSOR_MAP_SWIZZLE_64B);
}

// tw1: W1 with 128-row boxes (single-CTA kernel); tw1h: 64-row boxes (CTA-pair kernel)
// two (opj): th is the attention output o (the fused O-projection's A operand), two = W_o map
cudaError_t launch_mlp(const Opts& o, const CUtensorMap& th, const CUtensorMap& tw1, const CUtensorMap& tw1h,
                       const CUtensorMap& tw2, const MlpParams& p, int rows_for_grid, cudaStream_t s,
                       const CUtensorMap* tx = nullptr, const CUtensorMap* tln = nullptr,
                       const CUtensorMap* two = nullptr) {
  constexpr int smem = MlpSmem<256>::TOTAL;
  {
    cudaError_t e = ensure_smem_attr(mlp_tc_kernel<256, 1>, smem);
    if (e == cudaSuccess) e = ensure_smem_attr(mlp_tc_kernel<256, 2>, smem);
    if (e == cudaSuccess) e = ensure_smem_attr(mlp_tc_kernel<256, 1, true>, smem);
    if (e == cudaSuccess) e = ensure_smem_attr(mlp_tc_kernel<256, 2, true>, smem);
    if (e != cudaSuccess) return e;
  }
  const int tiles = (pad_rows(rows_for_grid, p.ln_cap > 0 ? p.ln_cap : rows_for_grid + 256) + 127) / 128;
  MlpParams q = p;
  q.staged = (tx != nullptr && (tln != nullptr || p.ln_g == nullptr)) ? 1 : 0;
  const CUtensorMap& mx = tx ? *tx : th;
  const CUtensorMap& ml = tln ? *tln : th;
  // CTA pairs (cta_group::2 MMAs, each SM holding half of every weight operand) with the fused
  // O-projection only: without it (option 11 = 0) the pair kernel hung with >= 5 tiles per pair
  // (128 c640 frames) and the single-CTA kernel runs
  if (o.mlp_cluster && two && num_sms(o) >= 2) {
    const int pairs = (tiles + 1) / 2;
    const int clusters = std::max(1, std::min(pairs, num_sms(o) / 2));
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(2 * clusters);
    lc.blockDim = dim3(MLP_THREADS);
    lc.dynamicSmemBytes = smem;
    lc.stream = s;
    cudaLaunchAttribute la[1];
    la[0].id = cudaLaunchAttributeClusterDimension;
    la[0].val.clusterDim.x = 2;
    la[0].val.clusterDim.y = 1;
    la[0].val.clusterDim.z = 1;
    lc.attrs = la;
    lc.numAttrs = 1;
    cudaError_t e = two ? cudaLaunchKernelEx(&lc, mlp_tc_kernel<256, 2, true>, th, tw1h, tw2, q, mx, ml, *two)
                        : cudaLaunchKernelEx(&lc, mlp_tc_kernel<256, 2>, th, tw1h, tw2, q, mx, ml, th);
    ++g_launches;
    return e != cudaSuccess ? e : cudaGetLastError();
  }
  const int grid = std::max(1, balanced_grid(o, tiles, num_sms(o)));
  const cudaError_t le =
      two ? launch_ex(mlp_tc_kernel<256, 1, true>, dim3(grid), dim3(MLP_THREADS), smem, s, th, tw1, tw2, q, mx, ml, *two)
          : launch_ex(mlp_tc_kernel<256, 1>, dim3(grid), dim3(MLP_THREADS), smem, s, th, tw1, tw2, q, mx, ml, th);
  if (le != cudaSuccess) return le;
  ++g_launches;
  return cudaGetLastError();
}

template <int NPP, int SLEEP = 32, int NWG = 4>
cudaError_t launch_attn7_t(const Opts& o, const CUtensorMap& tq64, const CUtensorMap& tq32, const AttnParams& p,
                           int items_ub, int nh, int T,
                           cudaStream_t s) {
  auto kern = attn7_tc_kernel<NWG, NPP, SLEEP>;
  constexpr int smem = Attn7Smem<NWG>::TOTAL;
  if (cudaError_t e = ensure_smem_attr(kern, smem); e != cudaSuccess) return e;
  const int grid = std::max(1, std::min((items_ub + NWG - 1) / NWG, num_sms(o)));
  cudaError_t e = launch_ex(kern, dim3(grid), dim3(attn7_threads(NWG)), smem, s, tq64, tq32, p, T, nh);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess && getenv("CFD_VERBOSE")) {
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, kern);
    fprintf(stderr, "attention v7 launch (grid %d, %d threads, %d B smem; kernel: %d regs): %s\n", grid,
            attn7_threads(NWG), smem, fa.numRegs, cudaGetErrorString(e));
  }
  return e;
}

// tq: qkv map with 128-row boxes (v1, v4); tq64 / tq32: the same tensor with 64- / 32-row boxes (v7)
cudaError_t launch_attention(const Opts& o, const CUtensorMap& tq, const CUtensorMap& tq64, const CUtensorMap& tq32,
                             const AttnParams& p,
                             int max_qtiles, int nh, int T, cudaStream_t s) {
  probe_begin(PK_ATTN, s);
  cudaError_t e;
  if (o.attn_variant == 7 && T <= ATTN7_MAX_T) {
    const int items_ub = T * max_qtiles * nh;
    switch (o.attn_npp) {
      case 0: e = launch_attn7_t<0>(o, tq64, tq32, p, items_ub, nh, T, s); break;
      case 6: e = launch_attn7_t<6>(o, tq64, tq32, p, items_ub, nh, T, s); break;
      case 8: e = launch_attn7_t<8>(o, tq64, tq32, p, items_ub, nh, T, s); break;
      case 4: e = launch_attn7_t<4>(o, tq64, tq32, p, items_ub, nh, T, s); break;
      default:
        e = o.attn_nwg == 3       ? launch_attn7_t<2, 32, 3>(o, tq64, tq32, p, items_ub, nh, T, s)
            : o.attn_sleep == 0   ? launch_attn7_t<2, 0>(o, tq64, tq32, p, items_ub, nh, T, s)
            : o.attn_sleep == 1   ? launch_attn7_t<2, 1>(o, tq64, tq32, p, items_ub, nh, T, s)
            : o.attn_sleep == 2   ? launch_attn7_t<2, 2>(o, tq64, tq32, p, items_ub, nh, T, s)
            : o.attn_sleep == 8   ? launch_attn7_t<2, 8>(o, tq64, tq32, p, items_ub, nh, T, s)
            : o.attn_sleep == 128 ? launch_attn7_t<2, 128>(o, tq64, tq32, p, items_ub, nh, T, s)
                                  : launch_attn7_t<2, 32>(o, tq64, tq32, p, items_ub, nh, T, s);
        break;
    }
  } else {
    auto kern = attn_tc_kernel<32, 3>;
    constexpr int smem = AttnSmem<32, 3>::TOTAL;
    e = ensure_smem_attr(kern, smem);
    if (e != cudaSuccess) return e;
    kern<<<dim3(max_qtiles, nh, T), ATTN_THREADS, smem, s>>>(tq, p, tq);
    e = cudaGetLastError();
  }
  probe_end(PK_ATTN, s);
  ++g_launches;
  return e;
}

cudaError_t launch_score(const CUtensorMap& tq, const CUtensorMap& tq32, const ScoreParams& p, int B,
                         cudaStream_t s) {
  auto kern = score_tc_kernel<32>;
  const int smem = ScoreSmem<32>::total(p.n_coarse);
  if (cudaError_t e = ensure_smem_attr(kern, ScoreSmem<32>::total(4096)); e != cudaSuccess) return e;
  probe_begin(PK_SCORE, s);
  launch_ex(kern, dim3((p.n_coarse + 127) / 128, B), dim3(SCORE_THREADS), smem, s, tq, tq32, p);
  probe_end(PK_SCORE, s);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_layernorm(const Opts& o, int d, const float* x, const float* g, const float* b, __nv_bfloat16* y, int M,
                             const int* m_dev, int m_cap, float eps, int rows_for_grid, cudaStream_t s) {
  const int rows_pad = pad_rows(rows_for_grid, m_cap);
  int blocks = (rows_pad + 7) / 8;
  blocks = std::max(1, std::min(blocks, num_sms(o) * 16));
  probe_begin(PK_LN, s);
  switch (d) {
    case 64: launch_ex(layernorm_kernel<2>, dim3(blocks), dim3(256), 0, s, x, g, b, y, M, m_dev, m_cap, eps); break;
    case 128: launch_ex(layernorm_kernel<4>, dim3(blocks), dim3(256), 0, s, x, g, b, y, M, m_dev, m_cap, eps); break;
    case 256: launch_ex(layernorm_kernel<8>, dim3(blocks), dim3(256), 0, s, x, g, b, y, M, m_dev, m_cap, eps); break;
    case 512: launch_ex(layernorm_kernel<16>, dim3(blocks), dim3(256), 0, s, x, g, b, y, M, m_dev, m_cap, eps); break;
    default: return cudaErrorInvalidValue;
  }
  probe_end(PK_LN, s);
  ++g_launches;
  return cudaGetLastError();
}

}  // namespace

// ====================================================================== ctx
struct LayerDev {
  uint16_t *wqkv, *wo, *w1, *w2;  // K-major [N, K]
  float *b_qkv, *b_o, *b_1, *b_2, *ln1_g, *ln1_b, *ln2_g, *ln2_b;
  CUtensorMap tm_qkv, tm_o, tm_1, tm_2;
  CUtensorMap tm_1c, tm_2c;  // W1 / W2 with 128-row x 64-k boxes (fused MLP ring slots)
  CUtensorMap tm_oc;         // W_o with 128-row x 64-k boxes (fused O-projection + MLP)
  CUtensorMap tm_1h;         // W1 with 64-row x 64-k boxes (CTA-pair fused MLP)
  CUtensorMap tm_qkv_h;      // W_qkv with 128-row x 64-k boxes (CTA-pair QKV: half a column block per CTA)
};

struct cfd_ctx {
  cfd_config cfg;
  Opts opt;  // tuning switches of this context (cfdx_set_option)
  int Nc, Nf, m, dh, Kc, Kf, gc_w, gf_w;
  void* block = nullptr;  // single device allocation for all ctx-owned data
  uint16_t *wc = nullptr, *wf = nullptr;
  float *bc = nullptr, *bf = nullptr, *pec = nullptr, *pef = nullptr;
  int* err = nullptr;
  std::vector<LayerDev> layers;
  CUtensorMap tm_wc, tm_wf;
  CUtensorMap tm_wc32;  // W_c with 32-k x 256-row SW64 boxes (image-sourced coarse embed)
  CUtensorMap tm_wc32h; // the same with 128-row boxes (CTA-pair embed: half the columns per CTA)
  bool has_wc32 = false;
  // NEXT f3 decoder (cfd_set_decoder): its own device block
  void* dec_block = nullptr;
  int dec_q = 0;
  float *dq0 = nullptr, *dlnq_g = nullptr, *dlnq_b = nullptr, *dlnm_g = nullptr, *dlnm_b = nullptr;
  uint16_t *dwq = nullptr, *dwkv = nullptr, *dwo = nullptr;  // K-major [N, K]
  float *dbq = nullptr, *dbkv = nullptr, *dbo = nullptr, *dwh = nullptr, *dbh = nullptr;
  CUtensorMap tm_dq, tm_dkv, tm_do;
};

namespace {

struct Workspace {
  __nv_bfloat16 *hbuf, *qkv, *obuf, *ff;
  uint16_t* patches;
  int32_t *frow, *fidx, *meta, *ccu;
  int32_t* attn_work;  // [2] attention work counter {claims, finished CTAs} of this workspace:
                       // zeroed by the first kernel of every call, reset by each attention
                       // launch's last CTA (so calls on different workspaces never share it)
  float* lse;
  int rows_cap;   // token capacity of hbuf/qkv/obuf/ff
  int lse_ld;
  size_t bytes;
};

// Carve the workspace for n tasks/frames.  base == nullptr -> size only.
Workspace carve(const cfd_ctx* c, int n, void* base) {
  Workspace w{};
  const cfd_config& g = c->cfg;
  // rows per task: Nf tokens, or the decoder's query count when larger (its cross-attention
  // output o has T * Q rows in obuf)
  const size_t rows = (size_t)n * std::max(c->Nf, c->dec_q) + 128;
  w.rows_cap = (int)rows;
  w.lse_ld = n * c->Nc;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align_up(off + bytes, 1024);
    return base ? static_cast<char*>(base) + o : nullptr;
  };
  w.hbuf = (__nv_bfloat16*)take(rows * g.d_model * 2);
  w.qkv = (__nv_bfloat16*)take(rows * 3 * g.d_model * 2);
  w.obuf = (__nv_bfloat16*)take(rows * g.d_model * 2);
  w.ff = (__nv_bfloat16*)take(rows * g.d_ff * 2);
  w.patches = (uint16_t*)take(((size_t)n * g.img_h * g.img_w * 3 + 128 * (size_t)c->Kc) * 2);
  w.frow = (int32_t*)take((size_t)n * c->Nf * 4 + 16);
  w.fidx = (int32_t*)take((size_t)n * c->Nf * 4 + 16);
  w.meta = (int32_t*)take(64);
  w.ccu = (int32_t*)take((size_t)(n + 1) * 4);
  w.attn_work = (int32_t*)take(16);
  w.lse = (float*)take((size_t)g.n_heads * n * c->Nc * 4 + 16);
  w.bytes = off;
  return w;
}

#define CFD_CUDA(x)                                  \
  do {                                               \
    cudaError_t e__ = (x);                           \
    if (e__ != cudaSuccess) return CFD_E_CUDA;       \
  } while (0)

// One pre-LN encoder block on the packed residual stream x (fp32 [*, d]).
// On entry w.hbuf must hold LN1(x) of this layer (bf16, pad rows zeroed): the
// first layer's comes from a standalone LayerNorm launch, every later one from the
// previous layer's MLP2 epilogue (EPI_F32_RESID_LN).  LN2 is fused into the
// O-projection epilogue the same way.
cfd_status run_layer(cfd_ctx* c, int l, float* x, int x_cap, int M_static, const int* m_dev, int rows_grid,
                     const int32_t* cu, int T, int max_qtiles, Workspace& w, bool want_lse, float* scores,
                     int score_B, cudaStream_t s, bool ln1_ready = false, const int32_t* kv_len = nullptr) {
  const cfd_config& g = c->cfg;
  Opts o = c->opt;
  if (kv_len) o.attn_variant = 7;  // key masking (padded batch) is a v7 feature
  const int d = g.d_model, F = g.d_ff;
  const bool fuse_ln = pick_bn(d) == d;  // one GEMM tile spans a whole row
  LayerDev& L = c->layers[l];
  CUtensorMap ta_h, ta_o, ta_f, tq, tq64, tq32;
  if (!make_amap(&ta_h, w.hbuf, w.rows_cap, d) || !make_amap(&ta_o, w.obuf, w.rows_cap, d) ||
      !make_amap(&ta_f, w.ff, w.rows_cap, F) || !make_qkvmap(&tq, w.qkv, w.rows_cap, d) ||
      !make_qkvmap(&tq64, w.qkv, w.rows_cap, d, 64) || !make_qkvmap(&tq32, w.qkv, w.rows_cap, d, 32))
    return CFD_E_CUDA;
  if ((l == 0 && !ln1_ready) || !fuse_ln)  // LN1
    CFD_CUDA(launch_layernorm(o, d, x, L.ln1_g, L.ln1_b, w.hbuf, M_static, m_dev, w.rows_cap, g.ln_eps, rows_grid, s));
  // QKV
  GemmParams p{};
  p.M = M_static; p.m_dev = m_dev; p.m_cap = w.rows_cap; p.N = 3 * d; p.K = d; p.bias = L.b_qkv;
  p.out_bf16 = w.qkv;
  if (o.qkv_pair && o.gemm_bres && d == 256 && num_sms(o) >= 2 * (3 * d / 256)) {
    probe_begin(PK_QKV, s);
    const cudaError_t e = launch_qkv_pair(o, ta_h, L.tm_qkv_h, p, rows_grid, s);
    probe_end(PK_QKV, s);
    CFD_CUDA(e);
  } else {
    CFD_CUDA(launch_gemm(o, EPI_BF16_BIAS, ta_h, L.tm_qkv, p, rows_grid, s, PK_QKV));
  }
  // attention
  AttnParams ap{};
  ap.cu_seqlens = cu; ap.d_model = d; ap.out = w.obuf; ap.lse = want_lse ? w.lse : nullptr; ap.lse_ld = w.lse_ld;
  ap.scale_log2 = 1.4426950408889634f / std::sqrt((float)c->dh);
  ap.stagger = o.attn_stagger;
  ap.producer_sleep = o.attn_psleep;
  if (o.attn_dyn) ap.work_counter = w.attn_work;  // dynamic item claiming (per-workspace counter)
  ap.kv_len = kv_len;
  CFD_CUDA(launch_attention(o, tq, tq64, tq32, ap, max_qtiles, g.n_heads, T, s));
  if (want_lse && scores) {
    ScoreParams sp{};
    sp.n_coarse = c->Nc; sp.n_heads = g.n_heads; sp.d_model = d; sp.lse = w.lse; sp.lse_ld = w.lse_ld;
    sp.scale_log2 = ap.scale_log2; sp.scores = scores;
    CFD_CUDA(launch_score(tq, tq32, sp, score_B, s));
  }
  const bool staged_ok = fuse_ln && o.staged_epi && (d % 64 == 0);
  if (o.fuse_oproj && o.fused_mlp && staged_ok && d == 256 && F % 128 == 0) {
    // O projection + residual + LN2 fused into the MLP kernel (LN2 never leaves the SM)
    CUtensorMap tx, tln;
    if (!make_tmap(&tx, x, d, x_cap, d, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B, true) ||
        !make_tmap(&tln, w.hbuf, d, w.rows_cap, d, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B))
      return CFD_E_CUDA;
    MlpParams mp{};
    mp.M = M_static; mp.m_dev = m_dev; mp.F = F; mp.b1 = L.b_1; mp.b2 = L.b_2; mp.x = x; mp.ln_eps = g.ln_eps;
    mp.bo = L.b_o; mp.ln2_g = L.ln2_g; mp.ln2_b = L.ln2_b; mp.keep_x1 = o.keep_x1;
    mp.ln_cap = w.rows_cap;
    if (l + 1 < g.n_layers) {
      const LayerDev& Ln = c->layers[l + 1];
      mp.ln_g = Ln.ln1_g; mp.ln_b = Ln.ln1_b; mp.ln_out = w.hbuf;
    }
    probe_begin(PK_MLP1, s);
    CFD_CUDA(launch_mlp(o, ta_o, L.tm_1c, L.tm_1h, L.tm_2c, mp, rows_grid, s, &tx, &tln, &L.tm_oc));
    probe_end(PK_MLP1, s);
    return CFD_OK;
  }
  // O projection + residual (+ LN2 -> hbuf)
  p = GemmParams{};
  p.M = M_static; p.m_dev = m_dev; p.m_cap = x_cap; p.N = d; p.K = d; p.bias = L.b_o; p.out_f32 = x; p.ld_out = d;
  CUtensorMap tx, tln;  // staging maps: fp32 x [x_cap, d] and bf16 LN out, 32 x 32 boxes
  const bool staged = fuse_ln && o.staged_epi && (d % 64 == 0) &&
                      make_tmap(&tx, x, d, x_cap, d, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B, true) &&
                      make_tmap(&tln, w.hbuf, d, w.rows_cap, d, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B);
  if (fuse_ln) {
    p.ln_g = L.ln2_g; p.ln_b = L.ln2_b; p.ln_out = w.hbuf; p.ln_cap = w.rows_cap; p.ln_eps = g.ln_eps;
    CFD_CUDA(launch_gemm(o, EPI_F32_RESID_LN, ta_o, L.tm_o, p, rows_grid, s, PK_OPROJ, staged ? &tx : nullptr,
                         staged ? &tln : nullptr));
  } else {
    CFD_CUDA(launch_gemm(o, EPI_F32_RESID, ta_o, L.tm_o, p, rows_grid, s, PK_OPROJ));
    CFD_CUDA(launch_layernorm(o, d, x, L.ln2_g, L.ln2_b, w.hbuf, M_static, m_dev, w.rows_cap, g.ln_eps, rows_grid, s));
  }
  if (o.fused_mlp && fuse_ln && d == 256 && F % 128 == 0) {
    // fused MLP1 + GELU + MLP2 + residual (+ next LN1): the hidden activations stay on chip
    MlpParams mp{};
    mp.M = M_static; mp.m_dev = m_dev; mp.F = F; mp.b1 = L.b_1; mp.b2 = L.b_2; mp.x = x; mp.ln_eps = g.ln_eps;
    if (l + 1 < g.n_layers) {
      const LayerDev& Ln = c->layers[l + 1];
      mp.ln_g = Ln.ln1_g; mp.ln_b = Ln.ln1_b; mp.ln_out = w.hbuf; mp.ln_cap = w.rows_cap;
    }
    probe_begin(PK_MLP1, s);
    CFD_CUDA(launch_mlp(o, ta_h, L.tm_1c, L.tm_1h, L.tm_2c, mp, rows_grid, s, staged ? &tx : nullptr, staged ? &tln : nullptr));
    probe_end(PK_MLP1, s);
    return CFD_OK;
  }
  // MLP1 + GELU
  p = GemmParams{};
  p.M = M_static; p.m_dev = m_dev; p.m_cap = w.rows_cap; p.N = F; p.K = d; p.bias = L.b_1; p.out_bf16 = w.ff;
  CFD_CUDA(launch_gemm(o, EPI_BF16_BIAS_GELU, ta_h, L.tm_1, p, rows_grid, s, PK_MLP1));
  // MLP2 + residual (+ next layer's LN1 -> hbuf)
  p = GemmParams{};
  p.M = M_static; p.m_dev = m_dev; p.m_cap = x_cap; p.N = d; p.K = F; p.bias = L.b_2; p.out_f32 = x; p.ld_out = d;
  if (fuse_ln && l + 1 < g.n_layers) {
    const LayerDev& Ln = c->layers[l + 1];
    p.ln_g = Ln.ln1_g; p.ln_b = Ln.ln1_b; p.ln_out = w.hbuf; p.ln_cap = w.rows_cap; p.ln_eps = g.ln_eps;
    CFD_CUDA(launch_gemm(o, EPI_F32_RESID_LN, ta_f, L.tm_2, p, rows_grid, s, PK_MLP2));
  } else {
    CFD_CUDA(launch_gemm(o, EPI_F32_RESID, ta_f, L.tm_2, p, rows_grid, s, PK_MLP2));
  }
  return CFD_OK;
}

cfd_status validate_cfg(const cfd_config* g) {
  if (!g) return CFD_E_ARG;
  if (g->img_h <= 0 || g->img_w <= 0 || g->patch_coarse <= 0 || g->patch_fine <= 0 || g->d_model <= 0 ||
      g->n_heads <= 0 || g->n_layers <= 0 || g->d_ff <= 0 || g->max_tasks <= 0)
    return CFD_E_ARG;
  if (g->score_layer < 0 || g->score_layer >= g->n_layers) return CFD_E_ARG;
  if (g->img_h % g->patch_coarse || g->img_w % g->patch_coarse || g->patch_coarse % g->patch_fine ||
      g->d_model % g->n_heads)
    return CFD_E_SHAPE;
  if (g->d_model / g->n_heads != 32) return CFD_E_UNSUPPORTED;
  if (g->d_model != 64 && g->d_model != 128 && g->d_model != 256 && g->d_model != 512) return CFD_E_UNSUPPORTED;
  if (g->d_ff % 64 || g->d_ff > GEMM_MAX_N) return CFD_E_UNSUPPORTED;
  if ((3 * g->patch_fine * g->patch_fine) % 64 || (g->patch_fine * 3 * 2) % 16) return CFD_E_UNSUPPORTED;
  const int Nc = (g->img_h / g->patch_coarse) * (g->img_w / g->patch_coarse);
  if (Nc > 4096) return CFD_E_UNSUPPORTED;
  return CFD_OK;
}

}  // namespace

// ====================================================================== C ABI
extern "C" {

const char* cfd_version(void) { return "cfdetr-b200 0.1 (sm_100a, tcgen05/TMEM/TMA)"; }

const char* cfd_status_str(cfd_status s) {
  switch (s) {
    case CFD_OK: return "ok";
    case CFD_E_ARG: return "invalid argument";
    case CFD_E_SHAPE: return "invalid shape";
    case CFD_E_UNSUPPORTED: return "unsupported configuration";
    case CFD_E_CAPACITY: return "capacity exceeded";
    case CFD_E_CUDA: return "CUDA error";
    case CFD_E_DEVICE: return "device-side input error";
  }
  return "unknown status";
}

int64_t cfdx_launch_count(void) { return g_launches.load(); }

cfd_status cfdx_attn_trace(uint64_t* dst, int32_t n_words) {
#ifdef CFD_TRACE
  if (!dst || n_words < ATTN_TRACE_WORDS) return CFD_E_ARG;
  CFD_CUDA(cudaMemcpyFromSymbol(dst, g_attn_trace, sizeof(unsigned long long) * ATTN_TRACE_WORDS));
  return CFD_OK;
#else
  (void)dst;
  (void)n_words;
  return CFD_E_ARG;
#endif
}

cfd_status cfdx_mlp_trace(uint64_t* dst, int32_t n_words) {
#ifdef CFD_TRACE
  if (!dst || n_words < MLP_TRACE_WORDS) return CFD_E_ARG;
  CFD_CUDA(cudaMemcpyFromSymbol(dst, g_mlp_trace, sizeof(unsigned long long) * MLP_TRACE_WORDS));
  return CFD_OK;
#else
  (void)dst;
  (void)n_words;
  return CFD_E_ARG;
#endif
}

cfd_status cfdx_probe_install(int32_t kind, void* const* h_start, void* const* h_end, int32_t capacity) {
  if (kind < 0 || kind >= kProbeKinds || capacity < 0 || (capacity > 0 && (!h_start || !h_end))) return CFD_E_ARG;
  Probe& p = g_probe[kind];
  p.start.assign(capacity, nullptr);
  p.end.assign(capacity, nullptr);
  for (int i = 0; i < capacity; ++i) {
    p.start[i] = static_cast<cudaEvent_t>(h_start[i]);
    p.end[i] = static_cast<cudaEvent_t>(h_end[i]);
  }
  p.count = 0;
  return CFD_OK;
}

cfd_status cfdx_set_option(cfd_ctx* ctx, int32_t key, int32_t value) {
  Opts& o = ctx ? ctx->opt : g_dbg_opts;
  const int b = value ? 1 : 0;
  switch (key) {
    case 0:
      if (value != 1 && value != 7) return CFD_E_ARG;
      o.attn_variant = value;
      return CFD_OK;
    case 1:
      if (value < 0 || value > 8 || (value & 1)) return CFD_E_ARG;
      o.attn_npp = value;
      return CFD_OK;
    case 2: o.fused_mlp = b; return CFD_OK;
    case 3: o.staged_epi = b; return CFD_OK;
    case 4: o.mlp_cluster = b; return CFD_OK;
    case 5:
      if (value < -2 || value > 100000) return CFD_E_ARG;  // -1 / -2: attention trace modes (debug library)
      o.attn_stagger = value;
      return CFD_OK;
    case 7: o.gemm_bres = b; return CFD_OK;
    case 11: o.fuse_oproj = b; return CFD_OK;
    case 13: o.embed_mode0 = b; return CFD_OK;
    case 14: o.embed_img = b; return CFD_OK;
    case 15: o.embed_ln = b; return CFD_OK;
    case 16: o.attn_dyn = b; return CFD_OK;
    case 17:
      if (value < 0 || value > 4096) return CFD_E_ARG;
      o.sm_cap = value;
      return CFD_OK;
    case 18: o.balanced_grid = b; return CFD_OK;
    case 19: o.keep_x1 = b; return CFD_OK;
    case 21:
      if (value != 0 && value != 1 && value != 2 && value != 8 && value != 32 && value != 128) return CFD_E_ARG;
      o.attn_sleep = value;
      return CFD_OK;
    case 22:
      if (value != 3 && value != 4) return CFD_E_ARG;
      o.attn_nwg = value;
      return CFD_OK;
    case 23: o.qkv_pair = b; return CFD_OK;
    case 25: o.embed_pair = b; return CFD_OK;
    case 24:
      if (value < 0 || value > 4096) return CFD_E_ARG;
      o.attn_psleep = value;
      return CFD_OK;
  }
  return CFD_E_ARG;
}

int32_t cfdx_probe_count(int32_t kind) {
  if (kind < 0 || kind >= kProbeKinds) return -1;
  return g_probe[kind].count;
}

cfd_status cfd_create(const cfd_config* cfg, const cfd_weights* wts, void* stream, cfd_ctx** out) {
  if (!out || !wts || !wts->h_layers || !wts->w_embed_c || !wts->w_embed_f || !wts->b_embed_c || !wts->b_embed_f ||
      !wts->pe_c || !wts->pe_f)
    return CFD_E_ARG;
  *out = nullptr;
  cfd_status st = validate_cfg(cfg);
  if (st != CFD_OK) return st;
  if (!get_encode_fn()) return CFD_E_CUDA;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cfd_ctx* c = new (std::nothrow) cfd_ctx();
  if (!c) return CFD_E_CUDA;
  c->cfg = *cfg;
  const cfd_config& g = *cfg;
  c->m = g.patch_coarse / g.patch_fine;
  c->gc_w = g.img_w / g.patch_coarse;
  c->gf_w = g.img_w / g.patch_fine;
  c->Nc = (g.img_h / g.patch_coarse) * c->gc_w;
  c->Nf = c->Nc * c->m * c->m;
  c->dh = g.d_model / g.n_heads;
  c->Kc = 3 * g.patch_coarse * g.patch_coarse;
  c->Kf = 3 * g.patch_fine * g.patch_fine;
  const int d = g.d_model, F = g.d_ff, L = g.n_layers;
  // sizes
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off = align_up(off + bytes, 256); return o; };
  const size_t o_wc = take((size_t)d * c->Kc * 2), o_wf = take((size_t)d * c->Kf * 2);
  const size_t o_bc = take(d * 4), o_bf = take(d * 4), o_pec = take((size_t)c->Nc * d * 4),
               o_pef = take((size_t)c->Nf * d * 4), o_err = take(16);
  std::vector<size_t> o_l(L);
  const size_t per_layer_mat = (size_t)(3 * d * d + d * d + d * F + F * d) * 2;
  const size_t per_layer_vec = (size_t)(3 * d + d + F + d + 4 * d) * 4;
  for (int l = 0; l < L; ++l) o_l[l] = take(per_layer_mat + per_layer_vec + 8 * 256);
  if (cudaMalloc(&c->block, off) != cudaSuccess) { delete c; return CFD_E_CUDA; }
  char* B = static_cast<char*>(c->block);
  c->wc = (uint16_t*)(B + o_wc); c->wf = (uint16_t*)(B + o_wf);
  c->bc = (float*)(B + o_bc); c->bf = (float*)(B + o_bf);
  c->pec = (float*)(B + o_pec); c->pef = (float*)(B + o_pef);
  c->err = (int*)(B + o_err);
  auto fail = [&](cfd_status e) { cudaFree(c->block); delete c; return e; };
  auto transpose = [&](const uint16_t* in, uint16_t* outp, int K, int N) {
    dim3 grid((N + 31) / 32, (K + 31) / 32);
    transpose_bf16_kernel<<<grid, dim3(32, 8), 0, s>>>(in, outp, K, N);
    ++g_launches;
    return cudaGetLastError();
  };
  if (transpose(wts->w_embed_c, c->wc, c->Kc, d) != cudaSuccess) return fail(CFD_E_CUDA);
  if (transpose(wts->w_embed_f, c->wf, c->Kf, d) != cudaSuccess) return fail(CFD_E_CUDA);
  if (cudaMemcpyAsync(c->bc, wts->b_embed_c, d * 4, cudaMemcpyDeviceToDevice, s) != cudaSuccess ||
      cudaMemcpyAsync(c->bf, wts->b_embed_f, d * 4, cudaMemcpyDeviceToDevice, s) != cudaSuccess ||
      cudaMemcpyAsync(c->pec, wts->pe_c, (size_t)c->Nc * d * 4, cudaMemcpyDeviceToDevice, s) != cudaSuccess ||
      cudaMemcpyAsync(c->pef, wts->pe_f, (size_t)c->Nf * d * 4, cudaMemcpyDeviceToDevice, s) != cudaSuccess ||
      cudaMemsetAsync(c->err, 0, 16, s) != cudaSuccess)
    return fail(CFD_E_CUDA);
  if (!make_wmap(&c->tm_wc, c->wc, d, c->Kc) || !make_wmap(&c->tm_wf, c->wf, d, c->Kf)) return fail(CFD_E_CUDA);
  c->has_wc32 = d == 256 && make_tmap(&c->tm_wc32, c->wc, c->Kc, d, c->Kc, 32, 256, CU_TENSOR_MAP_SWIZZLE_64B) &&
                make_tmap(&c->tm_wc32h, c->wc, c->Kc, d, c->Kc, 32, 128, CU_TENSOR_MAP_SWIZZLE_64B);
  c->layers.resize(L);
  for (int l = 0; l < L; ++l) {
    const cfd_layer_weights& hw = wts->h_layers[l];
    if (!hw.w_qkv || !hw.w_o || !hw.w_1 || !hw.w_2 || !hw.b_qkv || !hw.b_o || !hw.b_1 || !hw.b_2 || !hw.ln1_g ||
        !hw.ln1_b || !hw.ln2_g || !hw.ln2_b)
      return fail(CFD_E_ARG);
    LayerDev& ld = c->layers[l];
    char* p = B + o_l[l];
    size_t q = 0;
    auto sub = [&](size_t bytes) { char* r = p + q; q = align_up(q + bytes, 256); return r; };
    ld.wqkv = (uint16_t*)sub((size_t)3 * d * d * 2);
    ld.wo = (uint16_t*)sub((size_t)d * d * 2);
    ld.w1 = (uint16_t*)sub((size_t)d * F * 2);
    ld.w2 = (uint16_t*)sub((size_t)F * d * 2);
    ld.b_qkv = (float*)sub(3 * d * 4); ld.b_o = (float*)sub(d * 4); ld.b_1 = (float*)sub(F * 4);
    ld.b_2 = (float*)sub(d * 4); ld.ln1_g = (float*)sub(d * 4); ld.ln1_b = (float*)sub(d * 4);
    ld.ln2_g = (float*)sub(d * 4); ld.ln2_b = (float*)sub(d * 4);
    if (transpose(hw.w_qkv, ld.wqkv, d, 3 * d) != cudaSuccess || transpose(hw.w_o, ld.wo, d, d) != cudaSuccess ||
        transpose(hw.w_1, ld.w1, d, F) != cudaSuccess || transpose(hw.w_2, ld.w2, F, d) != cudaSuccess)
      return fail(CFD_E_CUDA);
    const std::pair<const float*, float*> vecs[] = {{hw.b_qkv, ld.b_qkv}, {hw.b_o, ld.b_o}, {hw.b_1, ld.b_1},
                                                    {hw.b_2, ld.b_2},     {hw.ln1_g, ld.ln1_g}, {hw.ln1_b, ld.ln1_b},
                                                    {hw.ln2_g, ld.ln2_g}, {hw.ln2_b, ld.ln2_b}};
    const size_t lens[] = {(size_t)3 * d, (size_t)d, (size_t)F, (size_t)d, (size_t)d, (size_t)d, (size_t)d, (size_t)d};
    for (int i = 0; i < 8; ++i)
      if (cudaMemcpyAsync(vecs[i].second, vecs[i].first, lens[i] * 4, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
        return fail(CFD_E_CUDA);
    if (!make_wmap(&ld.tm_qkv, ld.wqkv, 3 * d, d) || !make_wmap(&ld.tm_o, ld.wo, d, d) ||
        !make_wmap(&ld.tm_1, ld.w1, F, d) || !make_wmap(&ld.tm_2, ld.w2, d, F) ||
        !make_tmap(&ld.tm_1c, ld.w1, d, F, d, GEMM_BK, 128, CU_TENSOR_MAP_SWIZZLE_128B) ||
        !make_tmap(&ld.tm_2c, ld.w2, F, d, F, GEMM_BK, 128, CU_TENSOR_MAP_SWIZZLE_128B) ||
        !make_tmap(&ld.tm_1h, ld.w1, d, F, d, GEMM_BK, 64, CU_TENSOR_MAP_SWIZZLE_128B) ||
        !make_tmap(&ld.tm_oc, ld.wo, d, d, d, GEMM_BK, 128, CU_TENSOR_MAP_SWIZZLE_128B) ||
        !make_tmap(&ld.tm_qkv_h, ld.wqkv, d, 3 * d, d, GEMM_BK, 128, CU_TENSOR_MAP_SWIZZLE_128B))
      return fail(CFD_E_CUDA);
  }
  *out = c;
  return CFD_OK;
}

cfd_status cfd_destroy(cfd_ctx* c) {
  if (!c) return CFD_OK;
  // the caller guarantees no enqueued work still uses ctx (cfdetr.h); cudaFree itself waits
  // for the device to be idle before releasing the block
  cudaFree(c->block);
  if (c->dec_block) cudaFree(c->dec_block);
  delete c;
  return CFD_OK;
}

cfd_status cfd_query(const cfd_ctx* c, int32_t n, int32_t* h_Nc, int32_t* h_Nf, int32_t* h_max_tokens,
                     size_t* h_ws) {
  if (!c || n < 0) return CFD_E_ARG;
  if (h_Nc) *h_Nc = c->Nc;
  if (h_Nf) *h_Nf = c->Nf;
  if (h_max_tokens) *h_max_tokens = n * c->Nf;
  if (h_ws) *h_ws = carve(c, n > 0 ? n : 1, nullptr).bytes + 1024;
  return CFD_OK;
}

static void* align_ws(void* ws) {
  return reinterpret_cast<void*>(align_up(reinterpret_cast<uintptr_t>(ws), 1024));
}

cfd_status cfd_coarse_encode(cfd_ctx* c, int32_t B, const uint16_t* images, float* x0, float* y, float* scores,
                             float* layer_out, void* ws, size_t ws_bytes, void* stream) {
  if (!c) return CFD_E_ARG;
  if (B == 0) return CFD_OK;
  if (B < 0 || !images || !x0 || !y || !ws) return CFD_E_ARG;
  if (B > c->cfg.max_tasks) return CFD_E_CAPACITY;
  Workspace w = carve(c, B, align_ws(ws));
  if (w.bytes + 1024 > ws_bytes) return CFD_E_CAPACITY;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const cfd_config& g = c->cfg;
  const Opts& o = c->opt;
  const int d = g.d_model, M = B * c->Nc;
  probe_begin(PK_META, s);
  launch_ex(coarse_meta_kernel, dim3(1), dim3(256), 0, s, w.ccu, w.meta, B, c->Nc, w.attn_work);
  probe_end(PK_META, s);
  ++g_launches;
  CFD_CUDA(cudaGetLastError());
  GemmParams p{};
  p.M = M; p.m_cap = M; p.N = d; p.K = c->Kc; p.bias = c->bc; p.out_f32 = y; p.out2_f32 = x0; p.ld_out = d;
  p.pe = c->pec; p.pe_rows = c->Nc;
  // layer-0 LN1 fused into the embed epilogue (option 15): hbuf rows [0, M) here, the pad
  // rows [M, pad_rows) that attention tail tiles may read zeroed by a memset
  const bool ln0 = o.embed_ln && d == pick_bn(d);
  if (ln0) {
    const LayerDev& L0 = c->layers[0];
    p.ln_g = L0.ln1_g; p.ln_b = L0.ln1_b; p.ln_out = w.hbuf; p.ln_cap = w.rows_cap; p.ln_eps = g.ln_eps;
    const int pr = pad_rows(M, w.rows_cap);
    if (pr > M) CFD_CUDA(cudaMemsetAsync(w.hbuf + (size_t)M * d, 0, (size_t)(pr - M) * d * 2, s));
  }
  const int Pc = g.patch_coarse, gw = g.img_w / Pc, gh = g.img_h / Pc;
  // image-sourced embed: 3Pc-element segments split into 32-element k-blocks, whole coarse
  // rows per 128-row tile, box dims <= 256
  const bool img_ok = o.embed_img && d == 256 && (3 * Pc) % 32 == 0 && gw <= 128 && (128 / gw) <= 256 && c->has_wc32;
  if (img_ok) {
    CUtensorMap ti;
    p.img_gw = gw;
    p.img_rb = 128 / gw;
    p.img_thirds = 3 * Pc / 32;
    if (!make_img_map(&ti, images, B, g.img_h, g.img_w, Pc, p.img_rb)) return CFD_E_CUDA;
    probe_begin(PK_EMBED_C, s);
    cudaError_t e = o.embed_pair && num_sms(o) >= 2 ? launch_embed_pair(o, ti, c->tm_wc32h, p, M, s)
                                                    : launch_gemm_t<256, EPI_EMBED_COARSE, 3>(o, ti, c->tm_wc32, p, M, s,
                                                                                              nullptr, nullptr);
    probe_end(PK_EMBED_C, s);
    CFD_CUDA(e);
  } else {
    {
      const long long vec = (long long)B * g.img_h * (g.img_w / g.patch_coarse) * ((g.patch_coarse * 6) / 16);
      const int blocks = (int)std::min<long long>((vec + 255) / 256, (long long)num_sms(o) * 8);
      probe_begin(PK_IM2COL, s);
      launch_ex(im2col_kernel, dim3(blocks), dim3(256), 0, s, images, w.patches, B, g.img_h, g.img_w, g.patch_coarse);
      probe_end(PK_IM2COL, s);
      ++g_launches;
      CFD_CUDA(cudaGetLastError());
    }
    CUtensorMap ta;
    if (!make_amap(&ta, w.patches, M, c->Kc)) return CFD_E_CUDA;
    CFD_CUDA(launch_gemm(o, EPI_EMBED_COARSE, ta, c->tm_wc, p, M, s, PK_EMBED_C));
  }
  (void)gh;
  const int max_qtiles = (c->Nc + ATTN_BQ - 1) / ATTN_BQ;
  for (int l = 0; l < g.n_layers; ++l) {
    const bool sl = (l == g.score_layer);
    cfd_status st =
        run_layer(c, l, y, M, M, nullptr, M, w.ccu, B, max_qtiles, w, sl && scores, scores, B, s, ln0 && l == 0);
    if (st != CFD_OK) return st;
    if (layer_out)
      CFD_CUDA(cudaMemcpyAsync(layer_out + (size_t)l * M * d, y, (size_t)M * d * 4, cudaMemcpyDeviceToDevice, s));
  }
  return CFD_OK;
}

cfd_status cfd_select_regions(cfd_ctx* c, int32_t T, const float* scores, cfd_select_mode mode, const int32_t* h_k,
                              float threshold, int32_t* sel_idx, int32_t* sel_count, void* stream) {
  if (!c) return CFD_E_ARG;
  if (T == 0) return CFD_OK;
  if (T < 0 || !scores || !sel_idx || !sel_count) return CFD_E_ARG;
  if (mode != CFD_SELECT_TOPK && mode != CFD_SELECT_THRESHOLD) return CFD_E_ARG;
  if (mode == CFD_SELECT_TOPK) {
    if (!h_k) return CFD_E_ARG;
    for (int t = 0; t < T; ++t)
      if (h_k[t] < 0 || h_k[t] > c->Nc) return CFD_E_ARG;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int Nc = c->Nc;
  for (int t0 = 0; t0 < T; t0 += SELECT_CHUNK) {
    const int nt = std::min(SELECT_CHUNK, T - t0);
    SelectK ks;
    std::memset(&ks, 0, sizeof(ks));
    if (mode == CFD_SELECT_TOPK) std::memcpy(ks.k, h_k + t0, nt * sizeof(int));
    const float* sc = scores + (size_t)t0 * Nc;
    int32_t* si = sel_idx + (size_t)t0 * Nc;
    int32_t* cnt = sel_count + t0;
    probe_begin(PK_SELECT, s);
    if (Nc <= 512) launch_ex(select_kernel<512>, dim3(nt), dim3(512), 0, s, sc, Nc, (int)mode, ks, threshold, si, cnt);
    else if (Nc <= 1024) launch_ex(select_kernel<1024>, dim3(nt), dim3(512), 0, s, sc, Nc, (int)mode, ks, threshold, si, cnt);
    else if (Nc <= 2048) launch_ex(select_kernel<2048>, dim3(nt), dim3(512), 0, s, sc, Nc, (int)mode, ks, threshold, si, cnt);
    else launch_ex(select_kernel<4096>, dim3(nt), dim3(512), 0, s, sc, Nc, (int)mode, ks, threshold, si, cnt);
    probe_end(PK_SELECT, s);
    ++g_launches;
    CFD_CUDA(cudaGetLastError());
  }
  return CFD_OK;
}

static cfd_status launch_gather(cfd_ctx* c, int T, const uint16_t* images, const float* x0, const int32_t* sel_idx,
                                const int32_t* sel_count, float* X, int32_t* cu, int32_t* msrc, uint16_t* A_f,
                                int32_t* frow, int32_t* fidx, int32_t* meta, int32_t* attn_work, cudaStream_t s,
                                int pad_stride = 0, int32_t* kv_len = nullptr) {
  GatherParams gp{};
  const cfd_config& g = c->cfg;
  gp.T = T; gp.Nc = c->Nc; gp.gc_w = c->gc_w; gp.m = c->m; gp.gf_w = c->gf_w; gp.d = g.d_model;
  gp.H = g.img_h; gp.W = g.img_w; gp.Pf = g.patch_fine;
  gp.images = images; gp.x0 = x0; gp.sel_idx = sel_idx; gp.sel_count = sel_count; gp.X = X; gp.cu_seqlens = cu;
  gp.mixed_src = msrc; gp.A_f = A_f; gp.frow = frow; gp.fidx = fidx; gp.meta = meta; gp.err = c->err;
  gp.zero2 = attn_work;
  gp.pad_stride = pad_stride; gp.kv_len = kv_len;
  const int G = std::max(1, std::min(32, (c->Nc + 31) / 32));
  const size_t smem = (size_t)2 * c->Nc * sizeof(int32_t);
  probe_begin(PK_GATHER, s);
  launch_ex(gather_kernel, dim3(T, G), dim3(256), smem, s, gp);
  probe_end(PK_GATHER, s);
  ++g_launches;
  CFD_CUDA(cudaGetLastError());
  return CFD_OK;
}

static cfd_status batch_refine_impl(cfd_ctx* c, int32_t T, const uint16_t* images, const float* x0,
                                    const int32_t* sel_idx, const int32_t* sel_count, const int32_t* h_token_counts,
                                    float* y, int32_t* cu, int32_t* msrc, float* layer_out, void* ws, size_t ws_bytes,
                                    void* stream, int pad = 0, int32_t* kv_len = nullptr);

cfd_status cfd_batch_refine(cfd_ctx* c, int32_t T, const uint16_t* images, const float* x0, const int32_t* sel_idx,
                            const int32_t* sel_count, const int32_t* h_token_counts, float* y, int32_t* cu,
                            int32_t* msrc, float* layer_out, void* ws, size_t ws_bytes, void* stream) {
  return batch_refine_impl(c, T, images, x0, sel_idx, sel_count, h_token_counts, y, cu, msrc, layer_out, ws, ws_bytes,
                           stream);
}

cfd_status cfd_batch_refine_padded(cfd_ctx* c, int32_t T, const uint16_t* images, const float* x0,
                                   const int32_t* sel_idx, const int32_t* sel_count, int32_t max_tokens, float* y,
                                   int32_t* cu, int32_t* kv_len, int32_t* msrc, float* layer_out, void* ws,
                                   size_t ws_bytes, void* stream) {
  if (!c) return CFD_E_ARG;
  if (T == 0) return CFD_OK;
  if (!kv_len || max_tokens < c->Nc || max_tokens > c->Nf) return CFD_E_ARG;
  if (T > ATTN7_MAX_T) return CFD_E_UNSUPPORTED;
  return batch_refine_impl(c, T, images, x0, sel_idx, sel_count, nullptr, y, cu, msrc, layer_out, ws, ws_bytes, stream,
                           max_tokens, kv_len);
}

static cfd_status batch_refine_impl(cfd_ctx* c, int32_t T, const uint16_t* images, const float* x0,
                                    const int32_t* sel_idx, const int32_t* sel_count, const int32_t* h_token_counts,
                                    float* y, int32_t* cu, int32_t* msrc, float* layer_out, void* ws, size_t ws_bytes,
                                    void* stream, int pad, int32_t* kv_len) {
  if (!c) return CFD_E_ARG;
  if (T == 0) return CFD_OK;
  if (T < 0 || !images || !x0 || !sel_idx || !sel_count || !y || !cu || !msrc || !ws) return CFD_E_ARG;
  if (T > c->cfg.max_tasks) return CFD_E_CAPACITY;
  Workspace w = carve(c, T, align_ws(ws));
  if (w.bytes + 1024 > ws_bytes) return CFD_E_CAPACITY;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const cfd_config& g = c->cfg;
  const int d = g.d_model;
  const int cap = pad > 0 ? T * pad : T * c->Nf;  // rows of y (and of each layer_out slice)
  // host-side sizing hints (grid sizes only; every kernel reads the true counts on device)
  int rows_grid = cap, fine_grid = cap;
  if (h_token_counts) {
    long long tot = 0;
    for (int t = 0; t < T; ++t) {
      const int n = h_token_counts[t];
      if (n < c->Nc || n > c->Nf || (n - c->Nc) % (c->m * c->m - 1 > 0 ? c->m * c->m - 1 : 1)) return CFD_E_ARG;
      tot += n;
    }
    rows_grid = (int)tot;
    const int m2 = c->m * c->m;
    fine_grid = (m2 > 1) ? (int)((tot - (long long)T * c->Nc) / (m2 - 1) * m2) : 0;
  }
  if (pad > 0) {  // pad-to-max: every task spans `pad` rows
    rows_grid = T * pad;
    fine_grid = (c->m * c->m > 1) ? T * (pad - c->Nc) / (c->m * c->m - 1) * (c->m * c->m) : 0;
  }
  cfd_status st = launch_gather(c, T, images, x0, sel_idx, sel_count, y, cu, msrc, w.patches, w.frow, w.fidx,
                                w.meta, w.attn_work, s, pad, kv_len);
  if (st != CFD_OK) return st;
  CUtensorMap ta;
  if (!make_amap(&ta, w.patches, cap + 128, c->Kf)) return CFD_E_CUDA;
  GemmParams p{};
  p.M = 0; p.m_dev = w.meta + 1; p.m_cap = cap; p.N = d; p.K = c->Kf; p.bias = c->bf; p.out_f32 = y; p.ld_out = d;
  p.pe = c->pef; p.pe_rows = c->Nf; p.frow = w.frow; p.fidx = w.fidx;
  CFD_CUDA(launch_gemm(c->opt, EPI_EMBED_FINE, ta, c->tm_wf, p, std::max(fine_grid, 1), s, PK_EMBED_F));
  const int max_qtiles = ((pad > 0 ? pad : c->Nf) + ATTN_BQ - 1) / ATTN_BQ;
  // padded batch: the attention never writes the pad rows of a split tail tile (rows past the
  // first 32 of a tile with <= 32 real rows, attn7_tc.cuh), so they stay zero from here
  if (pad > 0) CFD_CUDA(cudaMemsetAsync(w.obuf, 0, (size_t)w.rows_cap * d * sizeof(__nv_bfloat16), s));
  for (int l = 0; l < g.n_layers; ++l) {
    st = run_layer(c, l, y, cap, 0, w.meta, std::max(rows_grid, 1), cu, T, max_qtiles, w, false, nullptr, 0, s,
                   false, kv_len);
    if (st != CFD_OK) return st;
    if (layer_out)
      CFD_CUDA(cudaMemcpyAsync(layer_out + (size_t)l * cap * d, y, (size_t)cap * d * 4, cudaMemcpyDeviceToDevice, s));
  }
  return CFD_OK;
}

cfd_status cfd_refine_encode(cfd_ctx* c, const uint16_t* image, const float* x0, const int32_t* sel_idx,
                             const int32_t* sel_count, float* y, int32_t* msrc, int32_t* cu, float* layer_out,
                             void* ws, size_t ws_bytes, void* stream) {
  return cfd_batch_refine(c, 1, image, x0, sel_idx, sel_count, nullptr, y, cu, msrc, layer_out, ws, ws_bytes,
                          stream);
}

// ------------------------------------------------------------------ NEXT f3: decoder
cfd_status cfd_set_decoder(cfd_ctx* c, const cfd_decoder_weights* dw, void* stream) {
  if (!c || !dw || !dw->queries || !dw->ln_q_g || !dw->ln_q_b || !dw->ln_m_g || !dw->ln_m_b || !dw->w_q ||
      !dw->w_kv || !dw->w_o || !dw->b_q || !dw->b_kv || !dw->b_o || !dw->w_head || !dw->b_head)
    return CFD_E_ARG;
  if (dw->n_queries <= 0 || dw->n_queries > 128) return CFD_E_ARG;
  if (c->dh != 32 || pick_bn(c->cfg.d_model) != c->cfg.d_model) return CFD_E_UNSUPPORTED;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int d = c->cfg.d_model, Q = dw->n_queries;
  if (c->dec_block) {
    cudaStreamSynchronize(s);
    cudaFree(c->dec_block);
    c->dec_block = nullptr;
  }
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off = align_up(off + bytes, 256); return o; };
  const size_t o_q0 = take((size_t)Q * d * 4), o_ln = take((size_t)4 * d * 4), o_wq = take((size_t)d * d * 2),
               o_wkv = take((size_t)2 * d * d * 2), o_wo = take((size_t)d * d * 2), o_b = take((size_t)4 * d * 4),
               o_wh = take((size_t)d * 5 * 4 + 5 * 4);
  if (cudaMalloc(&c->dec_block, off) != cudaSuccess) return CFD_E_CUDA;
  char* B = static_cast<char*>(c->dec_block);
  c->dec_q = Q;
  c->dq0 = (float*)(B + o_q0);
  c->dlnq_g = (float*)(B + o_ln); c->dlnq_b = c->dlnq_g + d; c->dlnm_g = c->dlnq_b + d; c->dlnm_b = c->dlnm_g + d;
  c->dwq = (uint16_t*)(B + o_wq); c->dwkv = (uint16_t*)(B + o_wkv); c->dwo = (uint16_t*)(B + o_wo);
  c->dbq = (float*)(B + o_b); c->dbkv = c->dbq + d; c->dbo = c->dbkv + 2 * d;
  c->dwh = (float*)(B + o_wh); c->dbh = c->dwh + (size_t)d * 5;
  auto cp = [&](void* dst, const void* src, size_t bytes) {
    return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, s) == cudaSuccess;
  };
  auto transpose = [&](const uint16_t* in, uint16_t* outp, int K, int N) {
    dim3 grid((N + 31) / 32, (K + 31) / 32);
    transpose_bf16_kernel<<<grid, dim3(32, 8), 0, s>>>(in, outp, K, N);
    ++g_launches;
    return cudaGetLastError() == cudaSuccess;
  };
  if (!cp(c->dq0, dw->queries, (size_t)Q * d * 4) || !cp(c->dlnq_g, dw->ln_q_g, d * 4) ||
      !cp(c->dlnq_b, dw->ln_q_b, d * 4) || !cp(c->dlnm_g, dw->ln_m_g, d * 4) || !cp(c->dlnm_b, dw->ln_m_b, d * 4) ||
      !cp(c->dbq, dw->b_q, d * 4) || !cp(c->dbkv, dw->b_kv, 2 * d * 4) || !cp(c->dbo, dw->b_o, d * 4) ||
      !cp(c->dwh, dw->w_head, (size_t)d * 5 * 4) || !cp(c->dbh, dw->b_head, 5 * 4) ||
      !transpose(dw->w_q, c->dwq, d, d) || !transpose(dw->w_kv, c->dwkv, d, 2 * d) || !transpose(dw->w_o, c->dwo, d, d))
    return CFD_E_CUDA;
  if (!make_wmap(&c->tm_dq, c->dwq, d, d) || !make_wmap(&c->tm_dkv, c->dwkv, 2 * d, d) ||
      !make_wmap(&c->tm_do, c->dwo, d, d))
    return CFD_E_CUDA;
  return CFD_OK;
}

cfd_status cfd_decode(cfd_ctx* c, int32_t T, const float* y, const int32_t* cu, int32_t max_tokens, float* z,
                      float* boxes, float* conf, void* ws, size_t ws_bytes, void* stream) {
  if (!c) return CFD_E_ARG;
  if (T == 0) return CFD_OK;
  if (T < 0 || !y || !cu || !boxes || !conf || !ws || max_tokens <= 0 || !c->dec_block) return CFD_E_ARG;
  if (T > c->cfg.max_tasks) return CFD_E_CAPACITY;
  Workspace w = carve(c, T, align_ws(ws));
  if (w.bytes + 1024 > ws_bytes || max_tokens > T * c->Nf) return CFD_E_CAPACITY;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const cfd_config& g = c->cfg;
  const int d = g.d_model, Q = c->dec_q, QR = T * Q;
  if ((size_t)QR + 128 > (size_t)w.rows_cap) return CFD_E_CAPACITY;  // obuf rows (carve sizes them)
  // workspace reuse: LN_m(y) -> hbuf, [k | v] -> qkv (2d columns), o -> obuf (T*Q rows),
  // LN_q(Q0) and q -> the ff region (256 rows each), z (if not requested) -> the patches region
  __nv_bfloat16* hq = w.ff;
  __nv_bfloat16* qb = w.ff + (size_t)256 * d;
  __nv_bfloat16* kvb = w.qkv;
  float* zz = z ? z : reinterpret_cast<float*>(w.patches);
  CUtensorMap tmhq, tmhm, tmq, tmkv, tmo;
  if (!make_amap(&tmhq, hq, 256, d) || !make_amap(&tmhm, w.hbuf, w.rows_cap, d) ||
      !make_tmap(&tmq, qb, d, 256, d, 32, 128, CU_TENSOR_MAP_SWIZZLE_64B) ||
      !make_tmap(&tmkv, kvb, 2 * d, w.rows_cap, 2 * d, 32, 128, CU_TENSOR_MAP_SWIZZLE_64B) ||
      !make_amap(&tmo, w.obuf, w.rows_cap, d))
    return CFD_E_CUDA;
  // queries: q = LN_q(Q0) W_q + b_q (rows >= Q zero / padding)
  const Opts& o = c->opt;
  CFD_CUDA(launch_layernorm(o, d, c->dq0, c->dlnq_g, c->dlnq_b, hq, Q, nullptr, 256, g.ln_eps, Q, s));
  GemmParams p{};
  p.M = Q; p.m_cap = 256; p.N = d; p.K = d; p.bias = c->dbq; p.out_bf16 = qb;
  CFD_CUDA(launch_gemm(o, EPI_BF16_BIAS, tmhq, c->tm_dq, p, Q, s));
  // memory: [k | v] = LN_m(y) W_kv + b_kv over the packed tokens (count cu[T] on the device)
  const int* m_dev = cu + T;
  CFD_CUDA(launch_layernorm(o, d, y, c->dlnm_g, c->dlnm_b, w.hbuf, max_tokens, m_dev, w.rows_cap, g.ln_eps, max_tokens, s));
  p = GemmParams{};
  p.M = max_tokens; p.m_dev = m_dev; p.m_cap = w.rows_cap; p.N = 2 * d; p.K = d; p.bias = c->dbkv; p.out_bf16 = kvb;
  CFD_CUDA(launch_gemm(o, EPI_BF16_BIAS, tmhm, c->tm_dkv, p, max_tokens, s));
  // cross-attention: one CTA per (head, task), the Q query rows against task t's tokens
  {
    auto kern = attn_tc_kernel<32, 3, true>;
    constexpr int smem = AttnSmem<32, 3>::TOTAL;
    CFD_CUDA(ensure_smem_attr(kern, smem));
    AttnParams ap{};
    ap.cu_seqlens = cu; ap.d_model = d; ap.out = w.obuf; ap.n_q = Q;
    ap.scale_log2 = 1.4426950408889634f / std::sqrt((float)c->dh);
    kern<<<dim3(1, g.n_heads, T), ATTN_THREADS, smem, s>>>(tmq, ap, tmkv);
    ++g_launches;
    CFD_CUDA(cudaGetLastError());
  }
  // z = Q0 + o W_o + b_o
  {
    const long long vec = (long long)QR * d / 4;
    const int blocks = (int)std::min<long long>((vec + 255) / 256, (long long)num_sms(o) * 4);
    launch_ex(broadcast_rows_kernel, dim3(blocks), dim3(256), 0, s, c->dq0, zz, T, Q, d);
    ++g_launches;
    CFD_CUDA(cudaGetLastError());
  }
  p = GemmParams{};
  p.M = QR; p.m_cap = w.rows_cap; p.N = d; p.K = d; p.bias = c->dbo; p.out_f32 = zz; p.ld_out = d;
  CFD_CUDA(launch_gemm(o, EPI_F32_RESID, tmo, c->tm_do, p, QR, s));
  // heads: [box | c] = sigmoid(z W_head + b_head)
  launch_ex(detect_heads_kernel, dim3((QR + 7) / 8), dim3(256), 0, s, zz, c->dwh, c->dbh, boxes, conf, QR, d);
  ++g_launches;
  CFD_CUDA(cudaGetLastError());
  return CFD_OK;
}

cfd_status cfd_hardness(cfd_ctx* c, int32_t B, int32_t Q, const float* conf, float c_hi, float tau,
                        int32_t* hard, void* stream) {
  if (!c) return CFD_E_ARG;
  if (B == 0) return CFD_OK;
  if (B < 0 || Q < 0 || !conf || !hard) return CFD_E_ARG;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  launch_ex(hardness_kernel, dim3((B + 127) / 128), dim3(128), 0, s, conf, B, Q, c_hi, tau, hard);
  ++g_launches;
  CFD_CUDA(cudaGetLastError());
  return CFD_OK;
}

cfd_status cfd_box_scores(cfd_ctx* c, int32_t B, int32_t Q, const float* boxes, const float* conf, float c_lo,
                          float c_hi, float* scores, void* stream) {
  if (!c) return CFD_E_ARG;
  if (B == 0) return CFD_OK;
  if (B < 0 || Q < 0 || Q > 4096 || !boxes || !conf || !scores) return CFD_E_ARG;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const cfd_config& g = c->cfg;
  launch_ex(box_scores_kernel, dim3(B), dim3(256), (size_t)std::max(Q, 1) * sizeof(int4), s,
           boxes, conf, Q, g.img_h, g.img_w, g.patch_coarse, c->gc_w, c->Nc, c_lo, c_hi, scores);
  ++g_launches;
  CFD_CUDA(cudaGetLastError());
  return CFD_OK;
}

static cfd_status launch_frames_u8(long long n, const uint8_t* src, const float* scale, const float* shift,
                                   uint16_t* dst, cudaStream_t s) {
  if (n == 0) return CFD_OK;
  if (n < 0 || !src || !dst || !scale || !shift) return CFD_E_ARG;
  FrameAffine a;
  for (int i = 0; i < 3; ++i) { a.scale[i] = scale[i]; a.shift[i] = shift[i]; }
  const long long units = std::max(n >> 4, 1LL);
  const int blocks = (int)std::min<long long>((units + 255) / 256, (long long)num_sms(g_dbg_opts) * 8);
  launch_ex(frames_u8_kernel, dim3(blocks), dim3(256), 0, s, src, dst, n, a);
  ++g_launches;
  CFD_CUDA(cudaGetLastError());
  return CFD_OK;
}

cfd_status cfd_frames_from_u8(cfd_ctx* c, int32_t n_frames, const uint8_t* src, const float* scale,
                              const float* shift, uint16_t* images, void* stream) {
  if (!c) return CFD_E_ARG;
  if (n_frames == 0) return CFD_OK;
  if (n_frames < 0) return CFD_E_ARG;
  const long long n = (long long)n_frames * c->cfg.img_h * c->cfg.img_w * 3;
  return launch_frames_u8(n, src, scale, shift, images, static_cast<cudaStream_t>(stream));
}

cfd_status cfdx_frames_u8(long long n, const uint8_t* src, const float* scale, const float* shift, uint16_t* dst,
                          void* stream) {
  return launch_frames_u8(n, src, scale, shift, dst, static_cast<cudaStream_t>(stream));
}

cfd_status cfd_check(cfd_ctx* c, void* stream) {
  if (!c) return CFD_E_ARG;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (cudaStreamSynchronize(s) != cudaSuccess) return CFD_E_CUDA;
  int e = 0;
  if (cudaMemcpy(&e, c->err, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess) return CFD_E_CUDA;
  if (e) {
    cudaMemset(c->err, 0, sizeof(int));
    return CFD_E_DEVICE;
  }
  return CFD_OK;
}

// ---------------------------------------------------------------------- debug entry points
cfd_status cfdx_gemm(int32_t M, int32_t N, int32_t K, const uint16_t* A, const uint16_t* W, const float* bias,
                     int32_t epi, uint16_t* out_bf16, float* out_f32, void* stream) {
  if (M <= 0 || N <= 0 || K <= 0 || N % 64 || K % 64 || N > GEMM_MAX_N || !A || !W || !bias) return CFD_E_ARG;
  if (epi < 0 || epi > 2 || (epi < 2 && !out_bf16) || (epi == 2 && !out_f32)) return CFD_E_ARG;
  CUtensorMap ta, tb;
  if (!make_amap(&ta, A, M, K) || !make_wmap(&tb, W, N, K)) return CFD_E_CUDA;
  GemmParams p{};
  p.M = M; p.m_cap = M; p.N = N; p.K = K; p.bias = bias; p.out_bf16 = (__nv_bfloat16*)out_bf16; p.out_f32 = out_f32;
  p.ld_out = N;
  CFD_CUDA(launch_gemm(g_dbg_opts, epi, ta, tb, p, M, static_cast<cudaStream_t>(stream)));
  return CFD_OK;
}

cfd_status cfdx_gemm_resid_ln(int32_t M, int32_t N, int32_t K, const uint16_t* A, const uint16_t* W,
                              const float* bias, float* x, const float* ln_g, const float* ln_b, float eps,
                              uint16_t* ln_out, int32_t ln_cap, int32_t staged, void* stream) {
  if (M <= 0 || N <= 0 || K <= 0 || N % 64 || K % 64 || N > GEMM_MAX_LN || !A || !W || !bias || !x || !ln_g ||
      !ln_b || !ln_out || ln_cap < M || pick_bn(N) != N)
    return CFD_E_ARG;
  CUtensorMap ta, tb, tx, tln;
  if (!make_amap(&ta, A, M, K) || !make_wmap(&tb, W, N, K) ||
      !make_tmap(&tx, x, N, M, N, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B, true) ||
      !make_tmap(&tln, ln_out, N, ln_cap, N, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B))
    return CFD_E_CUDA;
  GemmParams p{};
  p.M = M; p.m_cap = M; p.N = N; p.K = K; p.bias = bias; p.out_f32 = x; p.ld_out = N;
  p.ln_g = ln_g; p.ln_b = ln_b; p.ln_out = (__nv_bfloat16*)ln_out; p.ln_cap = ln_cap; p.ln_eps = eps;
  CFD_CUDA(launch_gemm(g_dbg_opts, EPI_F32_RESID_LN, ta, tb, p, M, static_cast<cudaStream_t>(stream), -1,
                       staged ? &tx : nullptr,
                       staged ? &tln : nullptr));
  return CFD_OK;
}

cfd_status cfdx_attention(int32_t T, const int32_t* cu, int32_t max_seqlen, int32_t rows_cap, int32_t d,
                          int32_t nh, const uint16_t* qkv, uint16_t* out, float* lse, int32_t lse_ld,
                          int32_t* work_counter, void* stream) {
  if (T <= 0 || !cu || !qkv || !out || max_seqlen <= 0 || rows_cap <= 0 || nh <= 0 || d % nh || d / nh != 32)
    return CFD_E_ARG;
  CUtensorMap tq, tq64, tq32;
  if (!make_qkvmap(&tq, qkv, rows_cap, d) || !make_qkvmap(&tq64, qkv, rows_cap, d, 64) ||
      !make_qkvmap(&tq32, qkv, rows_cap, d, 32))
    return CFD_E_CUDA;
  AttnParams ap{};
  ap.cu_seqlens = cu; ap.d_model = d; ap.out = (__nv_bfloat16*)out; ap.lse = lse; ap.lse_ld = lse_ld;
  ap.scale_log2 = 1.4426950408889634f / std::sqrt(32.0f);
  ap.stagger = g_dbg_opts.attn_stagger;
  ap.producer_sleep = g_dbg_opts.attn_psleep;
  // work_counter: caller-owned zeroed int[2] (dynamic claims, reset by the launch's last CTA)
  // or NULL (static round-robin); no state is shared between calls
  if (g_dbg_opts.attn_dyn) ap.work_counter = work_counter;
  CFD_CUDA(launch_attention(g_dbg_opts, tq, tq64, tq32, ap, (max_seqlen + ATTN_BQ - 1) / ATTN_BQ, nh, T, static_cast<cudaStream_t>(stream)));
  return CFD_OK;
}

cfd_status cfdx_layernorm(int32_t M, int32_t d, const float* x, const float* g, const float* b, float eps,
                          uint16_t* y, void* stream) {
  if (M <= 0 || !x || !g || !b || !y) return CFD_E_ARG;
  CFD_CUDA(launch_layernorm(g_dbg_opts, d, x, g, b, (__nv_bfloat16*)y, M, nullptr, M, eps, M,
                            static_cast<cudaStream_t>(stream)));
  return CFD_OK;
}

cfd_status cfdx_score(int32_t B, int32_t Nc, int32_t d, int32_t nh, const uint16_t* qkv, int32_t rows_cap,
                      const float* lse, int32_t lse_ld, float* scores, void* stream) {
  if (B <= 0 || Nc <= 0 || !qkv || !lse || !scores || d / nh != 32) return CFD_E_ARG;
  CUtensorMap tq, tq32;
  if (!make_qkvmap(&tq, qkv, rows_cap, d) || !make_qkvmap(&tq32, qkv, rows_cap, d, 32)) return CFD_E_CUDA;
  ScoreParams sp{};
  sp.n_coarse = Nc; sp.n_heads = nh; sp.d_model = d; sp.lse = lse; sp.lse_ld = lse_ld;
  sp.scale_log2 = 1.4426950408889634f / std::sqrt(32.0f); sp.scores = scores;
  CFD_CUDA(launch_score(tq, tq32, sp, B, static_cast<cudaStream_t>(stream)));
  return CFD_OK;
}

cfd_status cfdx_gather(cfd_ctx* c, int32_t T, const uint16_t* images, const float* x0, const int32_t* sel_idx,
                       const int32_t* sel_count, float* X, int32_t* cu, int32_t* msrc, uint16_t* A_f, int32_t* frow,
                       int32_t* fidx, int32_t* meta, void* stream) {
  if (!c || T <= 0 || !images || !x0 || !sel_idx || !sel_count || !X || !cu || !msrc || !A_f || !frow || !fidx ||
      !meta)
    return CFD_E_ARG;
  return launch_gather(c, T, images, x0, sel_idx, sel_count, X, cu, msrc, A_f, frow, fidx, meta, nullptr,
                       static_cast<cudaStream_t>(stream));
}

}  // extern "C"
