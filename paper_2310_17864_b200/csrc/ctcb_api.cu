// C ABI of the ctcb decoder (include/ctcb.h): argument checks, workspace
// layout, launch configuration.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <string>

#include "../../include/ctcb.h"
#include "ctcb_internal.h"

namespace ctcb {
__global__ void ctcb_decode_generic_kernel(const __grid_constant__ Params P);
__global__ void ctcb_decode_fast_kernel(const __grid_constant__ Params P);
__global__ void ctcb_decode_fast_pre_kernel(const __grid_constant__ Params P);
__global__ void ctcb_decode_fast_small_kernel(const __grid_constant__ Params P);
__global__ void ctcb_decode_fast_pre_small_kernel(const __grid_constant__ Params P);
__global__ void ctcb_decode_pair_kernel(const __grid_constant__ Params P);
__global__ void ctcb_decode_block_kernel(const __grid_constant__ Params P);
__global__ void ctcb_framemap_kernel(const __grid_constant__ Params P);
__global__ void ctcb_topk_kernel(const __grid_constant__ Params P);
__global__ void ctcb_rowoff_kernel(const __grid_constant__ Params P);
__global__ void ctcb_topk_wide_kernel(const __grid_constant__ Params P);
__global__ void ctcb_order_kernel(const int32_t* lens, int B, int32_t* order, int32_t* counter);
__global__ void ctcb_debug_kernel(const __grid_constant__ Params P, int32_t* out_topk_tok, float* out_topk_val,
                                  float* out_blank);
__global__ void ctcb_validate_kernel(const float* lp, long long sb, long long st, const int32_t* lens, int B,
                                     int T, int V, int strict, unsigned long long* out_key);
__global__ void ctcb_validate_decode_kernel(const unsigned long long* key, int T, int V, int64_t* out);
__global__ void ctcb_validate_post_kernel(const __grid_constant__ Params P);
}  // namespace ctcb

namespace ctcb {
// Zero-copy H2D gather for the host-buffer path: warps copy each utterance's
// valid frames straight from page-locked host memory (mapped into the device
// address space) into the dense device staging [B, T, V].  One launch per
// utterance range replaces one cudaMemcpyAsync per utterance (whose host-side
// enqueue cost, ~20 us each, bounded the copy rate); PCIe reads reach ~51 GB/s.
__global__ void __launch_bounds__(256) ctcb_gather_kernel(const float* __restrict__ src, long long sb, long long st,
                                                          const int32_t* __restrict__ lens, int b0, int b1, int T,
                                                          int Tp, int V, float* __restrict__ dst) {
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const bool vec = st == V && (V & 3) == 0 && (sb & 3) == 0 && (((uintptr_t)src) & 15) == 0;
  for (int b = b0 + ((blockIdx.x * blockDim.x + threadIdx.x) >> 5); b < b1; b += nw) {
    int n = lens[b];
    if (n <= 0) continue;
    if (n > T) n = T;
    const float* s = src + (size_t)b * sb;
    float* d = dst + (size_t)b * Tp * V;
    if (vec) {
      const float4* s4 = (const float4*)s;
      float4* d4 = (float4*)d;
      const long long m = (long long)n * V / 4;
      long long i = lane;
      for (; i + 96 < m; i += 128) {
        const float4 x0 = s4[i], x1 = s4[i + 32], x2 = s4[i + 64], x3 = s4[i + 96];
        d4[i] = x0; d4[i + 32] = x1; d4[i + 64] = x2; d4[i + 96] = x3;
      }
      for (; i < m; i += 32) d4[i] = s4[i];
    } else {
      for (int t = 0; t < n; t++)
        for (int v = lane; v < V; v += 32) d[(size_t)t * V + v] = s[(size_t)t * st + v];
    }
  }
}
}  // namespace ctcb

struct ctcb_handle;
namespace {
bool use_fast(const ctcb_handle* h);
}
struct ctcb_handle {
  int V, blank, beam, nbest, k, kpad, device;
  float cutoff;
  double beam_threshold;
  int num_sms, max_smem_optin;
  int merge_max;      // ctcb_set_merge_mode
  int tok_k;          // ctcb_set_beam_size_token (0: full vocabulary)
  int validate;       // ctcb_set_validate: 0 off, 1 strict (default), 2 without the norm check
  int force_generic;  // CTCB_FORCE_GENERIC=1: use the generic kernel for every beam (testing)
  unsigned long long* dbg;  // device [8] debug counters
  void* ws;
  size_t ws_bytes;
  // ctcb_decode_host staging (device): input, lens, outputs
  void* hbuf;
  size_t hbuf_bytes;
  cudaStream_t cstreams[4];  // H2D copy streams of ctcb_decode_host (lazy)
  cudaEvent_t cev[5];
  int have_cstreams;
  // ctcb_decode_host_async: per-chunk completion events and utterance ranges
  cudaEvent_t chunk_ev[64];
  int chunk_b0[64], chunk_b1[64];
  int n_chunks;
  // ctcb_kernel_timing: CUDA events around the beam kernel of each decode
  int timing;
  int n_timed;
  cudaEvent_t tev[2 * 64];
  int have_tev;
  const char* last_kernel;
  unsigned long long launches;  // kernels launched by this handle (ctcb_launch_count)
  // fused search (ctcb_set_lm / ctcb_set_silence)
  ctcb::LmTables lm;
  int has_lm;
  double lm_weight;
  int sil;
  double sil_score;
};

struct ctcb_lm {
  ctcb::LmModel* m;
};

namespace {

thread_local std::string g_last_error;
constexpr int kMaxChunks = 64;

bool use_fused(const ctcb_handle* h) { return h->has_lm || (h->sil >= 0 && h->sil_score != 0.0); }
bool use_fast(const ctcb_handle* h) { return h->beam <= ctcb::kFastBeam && !h->force_generic && !use_fused(h); }
// Fast kernel variant: compile-time layout when V <= kSmallV (ring 2, 2048-B rows).
bool fast_small(const ctcb::Params& P) {
  // (32-bit row offsets inside an utterance and utterance strides < 2^32 elements)
  return P.V <= ctcb::kSmallV && P.k <= 31 && P.bulk_ok && P.ring == 2 && P.row_bytes == ctcb::kSmallRowBytes &&
         P.tokK == 0 &&
         P.stride_b < (1ll << 32) && (long long)P.T_max * P.stride_t < (1ll << 32);
}
const void* fast_kernel_fn(const ctcb::Params& P, bool pre) {
  const bool sm = fast_small(P);
  if (pre) return sm ? (const void*)ctcb::ctcb_decode_fast_pre_small_kernel : (const void*)ctcb::ctcb_decode_fast_pre_kernel;
  return sm ? (const void*)ctcb::ctcb_decode_fast_small_kernel : (const void*)ctcb::ctcb_decode_fast_kernel;
}

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}
}  // namespace
namespace ctcb {
// Shared with the other translation units (ctcb_align.cu): record the message
// ctcb_last_error returns and pass the status through.
int set_error(int code, const char* msg) { return fail(code, msg); }
}  // namespace ctcb
namespace {
int cuda_fail(cudaError_t e, const char* where) {
  return fail(CTCB_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}
#define CTCB_CUDA(call)                               \
  do {                                                \
    cudaError_t e__ = (call);                         \
    if (e__ != cudaSuccess) return cuda_fail(e__, #call); \
  } while (0)

bool use_fast(const ctcb_handle* h);
// Precomputed-top-k mode for batches up to 10 utterances per SM: with few
// warps per SM the walk is latency-bound and the frame-parallel top-k keeps
// its per-frame latency off the chain (cfg4 shards of 512 / 1024 / 2048
// utterances: 2.95 / 3.32 / 4.06 ms vs 3.46 / 3.69 / 4.07 fused,
// tools/shard_modes.py); the full cfg4 batch (27 per SM) is faster fused.
// CTCB_TOPK_MODE=fused|precomp overrides.
bool use_precomp(const ctcb_handle* h, int B) {
  if (!use_fast(h)) return false;
  const char* m = getenv("CTCB_TOPK_MODE");
  if (m && strcmp(m, "fused") == 0) return false;
  if (m && strcmp(m, "precomp") == 0) return true;
  return B <= 10 * h->num_sms;
}

// Two utterances per warp (ctcb_pair.cu): the headline kernel for beam <= 16,
// V <= 512, blank 0, full vocabulary, 16-B aligned rows, large batches.
// CTCB_PAIR=0 disables it, CTCB_PAIR=1 forces it for any batch size.
bool use_pair(const ctcb_handle* h, const ctcb::Params& P, int B) {
  if (!use_fast(h) || h->tok_k != 0 || h->blank != 0 || h->V > ctcb::kSmallV || !P.bulk_ok) return false;
  const char* m = getenv("CTCB_PAIR");
  if (m && strcmp(m, "0") == 0) return false;
  if (m && strcmp(m, "1") == 0) return true;
  return false;  // opt-in while it is slower than the one-utterance-per-warp kernel
}

// One CTA per utterance for large beams (ctcb_block.cu): 16 < beam <= 128,
// V <= 2048, full vocabulary, no LM / silence bonus.  CTCB_BLOCK=0 disables it.
bool use_block(const ctcb_handle* h) {
  if (h->beam <= ctcb::kFastBeam || h->beam > ctcb::kBlockMaxBeam || h->V > ctcb::kBlockMaxV) return false;
  if (h->tok_k != 0 || h->force_generic || use_fused(h)) return false;
  const char* m = getenv("CTCB_BLOCK");
  return !(m && strcmp(m, "0") == 0);
}
// Block kernel with the top-k lists precomputed frame-parallel
// (ctcb_topk_wide_kernel): V <= 512.  CTCB_BLOCK_TOPK=inline keeps the
// in-kernel top-k.
bool use_block_pre(const ctcb_handle* h) {
  if (!use_block(h) || h->V > ctcb::kSmallV) return false;
  const char* m = getenv("CTCB_BLOCK_TOPK");
  return !(m && strcmp(m, "inline") == 0);
}

struct WsLayout {
  size_t frame_map, kept, trellis, order, counter, seqbuf, anc, topk_tok, topk_val, rowoff, ready, vkey, vdone, total;
};
WsLayout ws_layout(const ctcb_handle* h, int B, int T) {
  WsLayout w{};
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t r = ctcb::align_up(o, 256);
    o = r + bytes;
    return r;
  };
  w.frame_map = take((size_t)B * T * 4);
  w.kept = take((size_t)B * 4);
  w.trellis = take((size_t)B * T * h->beam * 4);
  w.order = take((size_t)B * 4);
  w.counter = take(4);
  w.seqbuf = take((size_t)B * 3 * (T + 1) * 4);
  w.anc = take((size_t)B * ((T + ctcb::kChunk - 1) / ctcb::kChunk) * 16);
  const size_t ntk = use_precomp(h, B) || use_block_pre(h) ? (size_t)B * T * h->k : 0;
  w.topk_tok = take(ntk * 4);
  w.topk_val = take(ntk * 4);
  w.rowoff = take(ntk ? ((size_t)B + 1) * 4 : 0);
  w.ready = take(use_precomp(h, B) || use_block_pre(h) ? (size_t)B * T * 4 : 0);
  w.vkey = take((size_t)B * 8);
  w.vdone = take((size_t)B * 4);
  w.total = ctcb::align_up(o, 256);
  return w;
}

int ring_for(int row_bytes) { (void)row_bytes; return 2; }

// Fill the launch parameters shared by the decode and debug kernels.
int make_params(ctcb_handle* h, const float* lp, int64_t sb, int64_t st, const int32_t* lens, int B, int T,
                void* ws, size_t ws_bytes, ctcb::Params& P, WsLayout& L) {
  if (!lp || !lens) return fail(CTCB_ERR_ARG, "log_probs and lens must be device pointers");
  if (B < 0 || T < 0) return fail(CTCB_ERR_ARG, "batch and t_max must be >= 0");
  if (st < h->V || sb < (int64_t)st * (T > 0 ? T : 1))
    return fail(CTCB_ERR_ARG, "strides must describe a [batch, t_max, vocab] layout with unit vocab stride");
  L = ws_layout(h, B, T);
  if (!ws) {
    if (h->ws_bytes < L.total) {
      if (h->ws) cudaFree(h->ws);
      h->ws = nullptr;
      h->ws_bytes = 0;
      CTCB_CUDA(cudaMalloc(&h->ws, L.total));
      h->ws_bytes = L.total;
    }
    ws = h->ws;
  } else if (ws_bytes < L.total) {
    return fail(CTCB_ERR_WORKSPACE, "workspace too small: need " + std::to_string(L.total) + " bytes");
  }
  char* base = (char*)ws;
  memset(&P, 0, sizeof(P));
  P.lp = lp;
  P.stride_b = sb;
  P.stride_t = st;
  P.lens = lens;
  P.B = B;
  P.T_max = T;
  P.V = h->V;
  P.blank = h->blank;
  P.beam = h->beam;
  P.nbest = h->nbest;
  P.k = h->k;
  P.kpad = h->kpad;
  P.cutoff = h->cutoff;
  P.skip = std::isfinite(h->cutoff) || h->cutoff < 0 ? 1 : 0;
  P.beam_threshold = h->beam_threshold;
  P.threshold_inf = std::isinf(h->beam_threshold) ? 1 : 0;
  P.merge_max = h->merge_max;
  P.tokK = h->tok_k;
  P.frame_map = (int32_t*)(base + L.frame_map);
  P.kept = (int32_t*)(base + L.kept);
  P.trellis = (uint32_t*)(base + L.trellis);
  P.order = (int32_t*)(base + L.order);
  P.counter = (int32_t*)(base + L.counter);
  P.seqbuf = (int32_t*)(base + L.seqbuf);
  P.anc = (uint8_t*)(base + L.anc);
  P.n_chunks = (T + ctcb::kChunk - 1) / ctcb::kChunk;
  P.topk_tok = (int32_t*)(base + L.topk_tok);
  P.topk_val = (float*)(base + L.topk_val);
  P.rowoff = (int32_t*)(base + L.rowoff);
  P.ready = nullptr;  // set by decode_impl when the top-k overlaps the walk
  P.validate = h->validate;
  P.vkey = (unsigned long long*)(base + L.vkey);
  P.vdone = (int32_t*)(base + L.vdone);
  // rows of V <= 512 are padded to 512 floats: the fast top-k reads 4 float4
  // chunks per lane without bounds checks (padding holds the sentinel)
  P.row_bytes = (int)ctcb::align_up((size_t)(h->V <= 512 ? 512 : h->V) * 4, 16);
  P.ring = ring_for(P.row_bytes);
  P.bulk_ok = ((uintptr_t)lp % 16 == 0) && ((h->V * 4) % 16 == 0) && ((st * 4) % 16 == 0) && ((sb * 4) % 16 == 0);
  return CTCB_OK;
}


// Overlapped precomputed mode: blocks per SM of ctcb_topk_kernel that fit
// beside the walk's own blocks (registers, shared memory, threads, block
// slots), so that both grids are resident at once and the walk consumes the
// lists while the top-k produces them.  0 = no room: the top-k runs first.
int topk_beside_walk(const ctcb_handle* h, const void* wfn, int wgrid, int wthreads, size_t wsmem, size_t tsmem,
                     int tthreads, int tbps, const void* tfn) {
  cudaFuncAttributes fw{}, ft{};
  if (cudaFuncGetAttributes(&fw, wfn) != cudaSuccess || cudaFuncGetAttributes(&ft, tfn) != cudaSuccess)
    return 0;
  int dev = 0, smem_sm = 0, regs_sm = 0, thr_sm = 0, blk_sm = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
  cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, dev);
  cudaDeviceGetAttribute(&thr_sm, cudaDevAttrMaxThreadsPerMultiProcessor, dev);
  cudaDeviceGetAttribute(&blk_sm, cudaDevAttrMaxBlocksPerMultiprocessor, dev);
  auto regs_of = [](int regs, int threads) -> long long {
    return (long long)((regs * 32 + 255) / 256 * 256) * ((threads + 31) / 32);
  };
  const long long wb = (wgrid + h->num_sms - 1) / h->num_sms, reserve = 1024;
  const long long smem_left = smem_sm - wb * ((long long)wsmem + (long long)fw.sharedSizeBytes + reserve);
  const long long regs_left = regs_sm - wb * regs_of(fw.numRegs, wthreads);
  const long long thr_left = thr_sm - wb * wthreads, blk_left = blk_sm - wb;
  long long fit = tbps;
  fit = std::min(fit, smem_left / ((long long)tsmem + (long long)ft.sharedSizeBytes + reserve));
  fit = std::min(fit, regs_left / regs_of(ft.numRegs, tthreads));
  fit = std::min(fit, thr_left / tthreads);
  fit = std::min(fit, blk_left);
  return fit > 0 ? (int)fit : 0;
}

// Choose the row-ring depth and warps per block: shared memory per warp must
// fit, then maximise resident warps per SM (occupancy API), and spread small
// batches over all SMs (at most ceil(B / num_sms) warps per block).
int launch_config(ctcb_handle* h, ctcb::Params& P, int B, bool fast) {
  const bool fused = use_fused(h);
  for (;;) {
    size_t total = fused ? ctcb::fused_smem_per_warp(P.beam, P.V, P.ring, P.row_bytes)
                   : fast ? ctcb::make_fast_layout(fast_small(P) ? ctcb::kSmallV : P.V, P.ring, P.row_bytes).total
                          : ctcb::make_layout(P.beam, P.kpad, P.V, P.ring, P.row_bytes).total;
    P.smem_per_warp = (int)total;
    if ((int)total <= h->max_smem_optin) break;
    if (P.ring > 1) { P.ring--; continue; }
    return fail(CTCB_ERR_UNSUPPORTED, "beam/vocabulary too large for one warp's shared memory");
  }
  const void* kfn = fused ? ctcb::fused_kernel_fn()
                    : fast ? fast_kernel_fn(P, use_precomp(h, B)) : (const void*)ctcb::ctcb_decode_generic_kernel;
  int max_wpb = h->max_smem_optin / P.smem_per_warp;
  max_wpb = max_wpb < 1 ? 1 : (max_wpb > 8 ? 8 : max_wpb);
  if (fused && max_wpb > 4) max_wpb = 4;  // __launch_bounds__(128)
  if (fast && max_wpb > 4) max_wpb = 4;  // fast kernel: __launch_bounds__(128, 6)
  int spread = (B + h->num_sms - 1) / h->num_sms;
  if (spread < 1) spread = 1;
  if (max_wpb > spread) max_wpb = spread;
  int best_wpb = 1, best_warps = -1;
  CTCB_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, h->max_smem_optin));
  for (int wpb = max_wpb; wpb >= 1; --wpb) {
    int bps = 0;
    CTCB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kfn, 32 * wpb, (size_t)P.smem_per_warp * wpb));
    if (bps * wpb > best_warps) { best_warps = bps * wpb; best_wpb = wpb; }
  }
  P.warps_per_block = best_wpb;
  return CTCB_OK;
}

}  // namespace

extern "C" {

const char* ctcb_status_string(int status) {
  switch (status) {
    case CTCB_OK: return "ok";
    case CTCB_ERR_ARG: return "invalid argument";
    case CTCB_ERR_CUDA: return "CUDA error";
    case CTCB_ERR_WORKSPACE: return "workspace too small";
    case CTCB_ERR_UNSUPPORTED: return "unsupported configuration";
    default: return "unknown status";
  }
}

const char* ctcb_last_error(void) { return g_last_error.c_str(); }

int ctcb_launch_count(ctcb_t* h, uint64_t* out) {
  if (!h || !out) return fail(CTCB_ERR_ARG, "NULL argument");
  *out = h->launches;
  return CTCB_OK;
}

int ctcb_debug_counters(ctcb_t* h, uint64_t* out8) {
  if (!h || !out8) return fail(CTCB_ERR_ARG, "NULL argument");
  memset(out8, 0, 8 * sizeof(uint64_t));
  if (!h->dbg) return CTCB_OK;
  CTCB_CUDA(cudaSetDevice(h->device));
  CTCB_CUDA(cudaMemcpy(out8, h->dbg, 8 * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  return CTCB_OK;
}

int ctcb_skip_cutoff(double thr, float* cutoff) {
  if (!cutoff) return fail(CTCB_ERR_ARG, "cutoff must not be NULL");
  if (!(thr > 0.0 && thr <= 1.0)) return fail(CTCB_ERR_ARG, "blank_skip_threshold must be in (0, 1]");
  if (thr == 1.0) { *cutoff = INFINITY; return CTCB_OK; }
  const double target = thr - 1e-12;  // emissions.py:29, :300-301
  if (!(target > 0.0)) { *cutoff = -INFINITY; return CTCB_OK; }
  auto drop = [&](float x) { return std::exp((double)x) >= target; };
  float c = (float)std::log(target);
  while (drop(std::nextafter(c, -INFINITY))) c = std::nextafter(c, -INFINITY);
  while (!drop(c)) c = std::nextafter(c, INFINITY);
  *cutoff = c;
  return CTCB_OK;
}

int ctcb_create(int V, int blank, int beam, int nbest, float skip_cutoff, double beam_threshold, int device,
                ctcb_t** out) {
  if (!out) return fail(CTCB_ERR_ARG, "out must not be NULL");
  *out = nullptr;
  if (V < 2) return fail(CTCB_ERR_ARG, "vocabulary must have at least 2 tokens (blank + 1)");
  if (V >= (1 << 22) - 1) return fail(CTCB_ERR_UNSUPPORTED, "vocabulary too large (max 4194302)");
  if (blank < 0 || blank >= V) return fail(CTCB_ERR_ARG, "blank_index " + std::to_string(blank) + " out of range");
  if (beam < 1) return fail(CTCB_ERR_ARG, "beam_size must be >= 1");
  if (beam > 512) return fail(CTCB_ERR_UNSUPPORTED, "beam_size must be <= 512");
  if (nbest < 1 || nbest > beam) return fail(CTCB_ERR_ARG, "n_best must be in [1, beam_size]");
  if (!(beam_threshold > 0)) return fail(CTCB_ERR_ARG, "beam_threshold must be positive");
  if (std::isnan(skip_cutoff)) return fail(CTCB_ERR_ARG, "skip_cutoff must not be NaN");
  int ndev = 0;
  CTCB_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(CTCB_ERR_ARG, "invalid CUDA device " + std::to_string(device));
  ctcb_handle* h = new ctcb_handle();
  h->V = V;
  h->blank = blank;
  h->beam = beam;
  h->nbest = nbest;
  h->k = 2 * beam < V - 1 ? 2 * beam : V - 1;
  h->kpad = ctcb::pow2_at_least(h->k);
  h->device = device;
  h->cutoff = skip_cutoff;
  h->beam_threshold = beam_threshold;
  h->ws = nullptr;
  h->ws_bytes = 0;
  h->dbg = nullptr;
  h->hbuf = nullptr;
  h->hbuf_bytes = 0;
  h->have_cstreams = 0;
  h->has_lm = 0;
  h->sil = -1;
  h->sil_score = 0.0;
  h->validate = 1;
  {
    const char* fg = getenv("CTCB_FORCE_GENERIC");
    h->force_generic = (fg && fg[0] == '1') ? 1 : 0;
  }
  cudaDeviceProp prop;
  cudaError_t e = cudaGetDeviceProperties(&prop, device);
  if (e != cudaSuccess) { delete h; return cuda_fail(e, "cudaGetDeviceProperties"); }
  if (prop.major < 10) { delete h; return fail(CTCB_ERR_UNSUPPORTED, "ctcb requires an sm_100 (Blackwell) GPU"); }
  h->num_sms = prop.multiProcessorCount;
  h->max_smem_optin = (int)prop.sharedMemPerBlockOptin;
  *out = h;
  return CTCB_OK;
}

int ctcb_set_merge_mode(ctcb_t* h, int max_mode) {
  if (!h) return fail(CTCB_ERR_ARG, "NULL handle");
  if (max_mode != 0 && max_mode != 1) return fail(CTCB_ERR_ARG, "merge mode must be 0 (logadd) or 1 (max)");
  h->merge_max = max_mode;
  return CTCB_OK;
}

int ctcb_set_validate(ctcb_t* h, int mode) {
  if (!h) return fail(CTCB_ERR_ARG, "NULL handle");
  if (mode < 0 || mode > 2) return fail(CTCB_ERR_ARG, "validate mode must be 0 (off), 1 (strict) or 2 (no norm check)");
  h->validate = mode;
  return CTCB_OK;
}

int ctcb_set_beam_size_token(ctcb_t* h, int K) {
  if (!h) return fail(CTCB_ERR_ARG, "NULL handle");
  if (K > h->V)
    return fail(CTCB_ERR_ARG, "beam_size_token " + std::to_string(K) + " exceeds vocabulary size " + std::to_string(h->V));
  h->tok_k = (K <= 0 || K >= h->V) ? 0 : K;
  return CTCB_OK;
}

int ctcb_kernel_timing(ctcb_t* h, int enable) {
  if (!h) return fail(CTCB_ERR_ARG, "NULL handle");
  CTCB_CUDA(cudaSetDevice(h->device));
  if (enable && !h->have_tev) {
    for (int i = 0; i < 2 * 64; i++) CTCB_CUDA(cudaEventCreate(&h->tev[i]));
    h->have_tev = 1;
  }
  h->timing = enable ? 1 : 0;
  h->n_timed = 0;
  return CTCB_OK;
}

int ctcb_kernel_time(ctcb_t* h, double* total_ms, int* launches, const char** kernel) {
  if (!h || !total_ms || !launches) return fail(CTCB_ERR_ARG, "NULL argument");
  *total_ms = 0.0;
  *launches = h->n_timed;
  if (kernel) *kernel = h->last_kernel ? h->last_kernel : "";
  if (!h->n_timed) return CTCB_OK;
  CTCB_CUDA(cudaSetDevice(h->device));
  CTCB_CUDA(cudaEventSynchronize(h->tev[2 * h->n_timed - 1]));
  for (int i = 0; i < h->n_timed; i++) {
    float ms = 0.f;
    CTCB_CUDA(cudaEventElapsedTime(&ms, h->tev[2 * i], h->tev[2 * i + 1]));
    *total_ms += ms;
  }
  return CTCB_OK;
}

int ctcb_destroy(ctcb_t* h) {
  if (!h) return CTCB_OK;
  if (h->has_lm) {
    cudaSetDevice(h->device);
    ctcb::lm_tables_free(&h->lm);
  }
  if (h->have_tev)
    for (int i = 0; i < 2 * 64; i++) cudaEventDestroy(h->tev[i]);
  if (h->ws) cudaFree(h->ws);
  if (h->dbg) cudaFree(h->dbg);
  if (h->hbuf) cudaFree(h->hbuf);
  if (h->have_cstreams) {
    for (int i = 0; i < 4; i++) cudaStreamDestroy(h->cstreams[i]);
    for (int i = 0; i < 5; i++) cudaEventDestroy(h->cev[i]);
    for (int i = 0; i < kMaxChunks; i++) cudaEventDestroy(h->chunk_ev[i]);
  }
  delete h;
  return CTCB_OK;
}

int ctcb_topk_size(const ctcb_t* h, int* k) {
  if (!h || !k) return fail(CTCB_ERR_ARG, "NULL argument");
  *k = h->k;
  return CTCB_OK;
}

int ctcb_workspace_bytes(const ctcb_t* h, int batch, int t_max, size_t* bytes) {
  if (!h || !bytes) return fail(CTCB_ERR_ARG, "NULL argument");
  if (batch < 0 || t_max < 0) return fail(CTCB_ERR_ARG, "batch and t_max must be >= 0");
  *bytes = ws_layout(h, batch, t_max).total;
  return CTCB_OK;
}

static int decode_impl(ctcb_t* h, const float* lp, int64_t sb, int64_t st, const int32_t* lens, int B, int T,
                       void* ws, size_t ws_bytes, void* stream, int32_t* out_tokens, int32_t* out_ts,
                       int32_t* out_len, double* out_score, int32_t* out_count, int32_t* out_status,
                       double* out_lm) {
  if (!h) return fail(CTCB_ERR_ARG, "NULL handle");
  if (!out_tokens || !out_len || !out_score || !out_count || !out_status)
    return fail(CTCB_ERR_ARG, "output pointers must not be NULL (out_timesteps may be)");
  if (B == 0) return CTCB_OK;
  CTCB_CUDA(cudaSetDevice(h->device));
  ctcb::Params P;
  WsLayout L;
  int rc = make_params(h, lp, sb, st, lens, B, T, ws, ws_bytes, P, L);
  if (rc) return rc;
  P.status = out_status;
  P.out_tokens = out_tokens;
  P.out_ts = out_ts;
  P.out_len = out_len;
  P.out_score = out_score;
  P.out_count = out_count;
  P.out_lm = out_lm;
  const bool fast = use_fast(h), fused = use_fused(h);
  if (fused) {
    P.lm_score = h->has_lm ? h->lm.score : nullptr;
    P.lm_next = h->lm.next;
    P.lm_fin = h->lm.fin;
    P.lm_wmax = h->lm.wmax;
    P.lm_wx = h->lm.wx;
    P.lm_A = h->lm.A;
    P.lm_wu = h->lm.wu;
    P.lm_xbits = h->lm.xbits;
    P.lm_start = h->lm.start;
    P.lm_weight = h->lm_weight;
  }
  P.sil = h->sil;
  P.sil_score = h->sil_score;
  rc = launch_config(h, P, B, fast);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  if (!h->dbg) CTCB_CUDA(cudaMalloc(&h->dbg, 8 * sizeof(unsigned long long)));
  CTCB_CUDA(cudaMemsetAsync(h->dbg, 0, 8 * sizeof(unsigned long long), s));
  P.dbg = h->dbg;
  if (P.validate) CTCB_CUDA(cudaMemsetAsync(P.vkey, 0xff, (size_t)B * 8, s));
  int n = 1;
  while (n < B) n <<= 1;
  size_t order_smem = n <= 8192 ? (size_t)n * 8 : 0;
  CTCB_CUDA(cudaFuncSetAttribute(ctcb::ctcb_order_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
  ctcb::ctcb_order_kernel<<<1, 1024, order_smem, s>>>(lens, B, P.order, P.counter);
  h->launches++;
  CTCB_CUDA(cudaGetLastError());
  const bool pair = use_pair(h, P, B);
  const bool pre = fast && !pair && use_precomp(h, B);
  const bool blk = use_block(h);
  if (pair) {  // 4 warps = 8 utterances per block, two halves' shared memory per warp
    P.smem_per_warp = (int)(2 * ctcb::make_pair_layout().total);
    P.warps_per_block = 4;
  }
  if (blk && use_block_pre(h)) {
    // frame maps -> top-k of every kept frame (one warp per row) -> beam walk
    P.precomp = 1;
    ctcb::ctcb_framemap_kernel<<<(B + 7) / 8, 256, 0, s>>>(P);
    h->launches++;
    CTCB_CUDA(cudaGetLastError());
  }
  if (blk) {  // one 256-thread CTA per utterance
    P.smem_per_warp = (int)ctcb::make_block_layout(ctcb::kBlockMaxBeam, 256, ctcb::kBlockMaxV, ctcb::kBlockMaxV * 4).total;
    P.warps_per_block = 8;
  }
  size_t smem = blk ? (size_t)P.smem_per_warp : (size_t)P.smem_per_warp * P.warps_per_block;
  const void* kfn = blk ? (const void*)ctcb::ctcb_decode_block_kernel
                    : pair ? (const void*)ctcb::ctcb_decode_pair_kernel
                    : fused ? ctcb::fused_kernel_fn()
                    : fast ? fast_kernel_fn(P, pre) : (const void*)ctcb::ctcb_decode_generic_kernel;
  CTCB_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int blocks_per_sm = 0;
  CTCB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, kfn, 32 * P.warps_per_block, smem));
  if (blocks_per_sm < 1) blocks_per_sm = 1;
  const int per_block = blk ? 1 : (pair ? 2 * P.warps_per_block : P.warps_per_block);
  int need = (B + per_block - 1) / per_block;
  if (blk) {
    // up to 2 utterances per SM: one CTA per SM walking the longest-first
    // queue beats two co-resident CTAs (the longest utterances set the time
    // and run ~25 % slower sharing an SM); CTCB_BLOCK_PER_SM overrides
    const int occ = blocks_per_sm;
    if (B <= 2 * h->num_sms) blocks_per_sm = 1;
    const char* m = getenv("CTCB_BLOCK_PER_SM");
    if (m && atoi(m) > 0) blocks_per_sm = atoi(m) < occ ? atoi(m) : occ;
  }
  int grid = h->num_sms * blocks_per_sm;
  if (grid > need) grid = need;
  // precomputed mode: frame maps -> top-k of every kept frame (frame-parallel)
  // -> beam walk.  When both grids fit on the SMs together, the top-k runs
  // frame-major beside the walk (the walk is its programmatic dependent and
  // waits per list on the ready flags); otherwise it runs first.
  bool overlap = false;
  ctcb::Params Q{};
  size_t tsmem = 0;
  int tk_grid = 0, tk_threads = 0;
  if (pre) {
    P.precomp = 1;
    ctcb::ctcb_framemap_kernel<<<(B + 7) / 8, 256, 0, s>>>(P);
    h->launches++;
    CTCB_CUDA(cudaGetLastError());
    Q = P;
    // V > 512 with 16-B rows: the top-k kernel reads rows from global memory
    // (no staging ring, row_bytes = 0), so far more warps fit per SM
    if (P.V > ctcb::kSmallV && P.bulk_ok && P.V % 4 == 0 && getenv("CTCB_TOPK_STAGED") == nullptr) Q.row_bytes = 0;
    Q.smem_per_warp = (int)ctcb::align_up((size_t)ctcb::kTopkRing * Q.row_bytes + 64 + 64 * 8 + 256 * 4 + 64 * 4 + 64 * 2, 128);
    int twpb = h->max_smem_optin / Q.smem_per_warp;
    twpb = twpb < 1 ? 1 : (twpb > 8 ? 8 : twpb);
    tsmem = (size_t)Q.smem_per_warp * twpb;
    tk_threads = 32 * twpb;
    CTCB_CUDA(cudaFuncSetAttribute(ctcb::ctcb_topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsmem));
    int tbps = 0;
    CTCB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&tbps, ctcb::ctcb_topk_kernel, tk_threads, tsmem));
    tk_grid = h->num_sms * (tbps > 0 ? tbps : 1);
    // default: overlap for V > 512 (rows from global memory: the top-k is
    // ~17 % of the sequential step at cfg3, and running it beside the walk
    // cuts the step by ~7 %); for V <= 512 the top-k is a few % of the step
    // and sharing the SMs slows the latency-bound walk by more than that
    // (cfg1 +0.5 %, 512- / 1,024-utterance shards +2 % / +11 %).
    // CTCB_OVERLAP=1 forces it, 0 disables it; CTCB_OVERLAP_BPS caps the
    // top-k blocks per SM.
    const char* ov = getenv("CTCB_OVERLAP");
    const char* ovb = getenv("CTCB_OVERLAP_BPS");
    const bool want = ov ? strcmp(ov, "0") != 0 : Q.row_bytes == 0;
    if (want) {
      int fit = topk_beside_walk(h, kfn, grid, 32 * P.warps_per_block, smem, tsmem, tk_threads, tbps,
                                 (const void*)ctcb::ctcb_topk_kernel);
      if (ovb && atoi(ovb) > 0 && atoi(ovb) < fit) fit = atoi(ovb);
      if (fit > 0) {
        overlap = true;
        tk_grid = h->num_sms * fit;
      }
    }
    if (overlap) {
      // both kernels prefer the largest shared-memory carve-out, so an SM
      // configured for one has room for the other
      CTCB_CUDA(cudaFuncSetAttribute(ctcb::ctcb_topk_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
      CTCB_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
      P.ready = (uint32_t*)((char*)P.topk_tok - L.topk_tok + L.ready);
      Q.ready = P.ready;
      CTCB_CUDA(cudaMemsetAsync(P.ready, 0, (size_t)B * T * 4, s));
    } else {
      ctcb::ctcb_rowoff_kernel<<<1, 1024, 0, s>>>(P);
      h->launches++;
      CTCB_CUDA(cudaGetLastError());
      Q.rowoff = P.rowoff;
      ctcb::ctcb_topk_kernel<<<tk_grid, tk_threads, tsmem, s>>>(Q);
      h->launches++;
      CTCB_CUDA(cudaGetLastError());
    }
  }
  // block kernel, precomputed lists (ctcb_topk_wide_kernel): beside the walk
  // as in the fast path (default; cfg2 beam 50 / 100: 9.80 -> 9.57 /
  // 15.14 -> 14.94 ms per step), or before it (CTCB_OVERLAP=0)
  bool overlap_blk = false;
  int tkw_grid = 0;
  if (blk && P.precomp) {
    int tbps = 0;
    CTCB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&tbps, ctcb::ctcb_topk_wide_kernel, 256, 0));
    tkw_grid = h->num_sms * (tbps > 0 ? tbps : 1);
    const char* ov = getenv("CTCB_OVERLAP");
    const char* ovb = getenv("CTCB_OVERLAP_BPS");
    if (!(ov && strcmp(ov, "0") == 0)) {
      int fit = topk_beside_walk(h, kfn, grid, 256, smem, 0, 256, tbps, (const void*)ctcb::ctcb_topk_wide_kernel);
      if (ovb && atoi(ovb) > 0 && atoi(ovb) < fit) fit = atoi(ovb);
      if (fit > 0) {
        overlap_blk = true;
        tkw_grid = h->num_sms * fit;
        CTCB_CUDA(cudaFuncSetAttribute(ctcb::ctcb_topk_wide_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        CTCB_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        P.ready = (uint32_t*)((char*)P.topk_tok - L.topk_tok + L.ready);
        CTCB_CUDA(cudaMemsetAsync(P.ready, 0, (size_t)B * T * 4, s));
      }
    }
    if (!overlap_blk) {
      ctcb::ctcb_rowoff_kernel<<<1, 1024, 0, s>>>(P);
      h->launches++;
      CTCB_CUDA(cudaGetLastError());
      ctcb::ctcb_topk_wide_kernel<<<tkw_grid, 256, 0, s>>>(P);
      h->launches++;
      CTCB_CUDA(cudaGetLastError());
    }
  }
  // diagnostics: CTCB_UTT_TRACE=path dumps a per-utterance timeline of the
  // fast kernels ([B, 2] uint64: smid << 48 | global warp, start ns; end ns)
  const char* trace_path = getenv("CTCB_UTT_TRACE");
  unsigned long long* trace = nullptr;
  if (trace_path && fast && !pair && !fused) {
    CTCB_CUDA(cudaMalloc(&trace, (size_t)B * 16 + 16 * 8));  // + phase cycle sums (-DCTCB_PHASES)
    CTCB_CUDA(cudaMemsetAsync(trace, 0, (size_t)B * 16 + 16 * 8, s));
    P.utt_trace = trace;
  }
  const bool timed = h->timing && h->n_timed < 64;
  if (timed) CTCB_CUDA(cudaEventRecord(h->tev[2 * h->n_timed], s));
  if (overlap) {  // the walk follows at once as its programmatic dependent
    ctcb::ctcb_topk_kernel<<<tk_grid, tk_threads, tsmem, s>>>(Q);
    h->launches++;
    CTCB_CUDA(cudaGetLastError());
  }
  if (overlap_blk) {
    ctcb::ctcb_topk_wide_kernel<<<tkw_grid, 256, 0, s>>>(P);
    h->launches++;
    CTCB_CUDA(cudaGetLastError());
  }
  if (blk) {
    void* args[] = {(void*)&P};
    if (overlap_blk) {
      cudaLaunchConfig_t lc{};
      lc.gridDim = dim3(grid);
      lc.blockDim = dim3(256);
      lc.dynamicSmemBytes = smem;
      lc.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      lc.attrs = at;
      lc.numAttrs = 1;
      CTCB_CUDA(cudaLaunchKernelExC(&lc, (const void*)ctcb::ctcb_decode_block_kernel, args));
    } else {
      CTCB_CUDA(cudaLaunchKernel((const void*)ctcb::ctcb_decode_block_kernel, dim3(grid), dim3(256), args, smem, s));
    }
    h->last_kernel = "ctcb_decode_block_kernel";
    h->launches++;
  } else if (pair) {
    void* args[] = {(void*)&P};
    CTCB_CUDA(cudaLaunchKernel((const void*)ctcb::ctcb_decode_pair_kernel, dim3(grid), dim3(32 * P.warps_per_block),
                               args, smem, s));
    h->last_kernel = "ctcb_decode_pair_kernel";
    h->launches++;
  } else if (fused) {
    void* args[] = {(void*)&P};
    CTCB_CUDA(cudaLaunchKernel(kfn, dim3(grid), dim3(32 * P.warps_per_block), args, smem, s));
    h->last_kernel = "ctcb_decode_fused_kernel";
    h->launches++;
  } else if (fast) {
    void* args[] = {(void*)&P};
    if (overlap) {
      cudaLaunchConfig_t lc{};
      lc.gridDim = dim3(grid);
      lc.blockDim = dim3(32 * P.warps_per_block);
      lc.dynamicSmemBytes = smem;
      lc.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      lc.attrs = at;
      lc.numAttrs = 1;
      CTCB_CUDA(cudaLaunchKernelExC(&lc, kfn, args));
    } else {
      CTCB_CUDA(cudaLaunchKernel(kfn, dim3(grid), dim3(32 * P.warps_per_block), args, smem, s));
    }
    h->last_kernel = !fast_small(P) ? (pre ? "ctcb_decode_fast_pre_kernel" : "ctcb_decode_fast_kernel")
                                    : (pre ? "ctcb_decode_fast_pre_small_kernel" : "ctcb_decode_fast_small_kernel");
    h->launches++;
  } else {
    ctcb::ctcb_decode_generic_kernel<<<grid, 32 * P.warps_per_block, smem, s>>>(P);
    h->last_kernel = "ctcb_decode_generic_kernel";
    h->launches++;
  }
  CTCB_CUDA(cudaGetLastError());
  if (timed) {
    CTCB_CUDA(cudaEventRecord(h->tev[2 * h->n_timed + 1], s));
    h->n_timed++;
  }
  if (trace) {
    std::vector<unsigned long long> buf((size_t)B * 2 + 16);
    CTCB_CUDA(cudaMemcpyAsync(buf.data(), trace, (size_t)B * 16 + 16 * 8, cudaMemcpyDeviceToHost, s));
    CTCB_CUDA(cudaStreamSynchronize(s));
    CTCB_CUDA(cudaFree(trace));
    if (FILE* f = fopen(trace_path, "wb")) {
      fwrite(buf.data(), 8, buf.size(), f);
      fclose(f);
    }
  }
  if (P.validate) {
    // rows the decode kernel did not screen (skipped frames, frames after a
    // dead beam, kernels without the fused check), then the per-utterance
    // verdict into out_status / out_len / out_count
    P.vfused = (blk || (fast && !pair && !fused)) ? 1 : 0;
    ctcb::ctcb_validate_post_kernel<<<(B + 7) / 8, 256, 0, s>>>(P);
    h->launches++;
    CTCB_CUDA(cudaGetLastError());
  }
  return CTCB_OK;
}

int ctcb_decode(ctcb_t* h, const float* lp, int64_t sb, int64_t st, const int32_t* lens, int B, int T, void* ws,
                size_t ws_bytes, void* stream, int32_t* out_tokens, int32_t* out_ts, int32_t* out_len,
                double* out_score, int32_t* out_count, int32_t* out_status) {
  return decode_impl(h, lp, sb, st, lens, B, T, ws, ws_bytes, stream, out_tokens, out_ts, out_len, out_score,
                     out_count, out_status, nullptr);
}

int ctcb_decode_lm(ctcb_t* h, const float* lp, int64_t sb, int64_t st, const int32_t* lens, int B, int T, void* ws,
                   size_t ws_bytes, void* stream, int32_t* out_tokens, int32_t* out_ts, int32_t* out_len,
                   double* out_score, double* out_lm, int32_t* out_count, int32_t* out_status) {
  return decode_impl(h, lp, sb, st, lens, B, T, ws, ws_bytes, stream, out_tokens, out_ts, out_len, out_score,
                     out_count, out_status, out_lm);
}

int ctcb_lm_create(int order, int64_t n_ngrams, const int32_t* words, const int32_t* lengths, const double* logprob,
                   const double* backoff, const int32_t* start, int start_len, int eos, int device, ctcb_lm_t** out) {
  if (!out) return fail(CTCB_ERR_ARG, "out must not be NULL");
  *out = nullptr;
  int ndev = 0;
  CTCB_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(CTCB_ERR_ARG, "invalid CUDA device " + std::to_string(device));
  ctcb::LmModel* m = nullptr;
  const char* err = "";
  int rc = ctcb::lm_model_create(order, n_ngrams, words, lengths, logprob, backoff, start, start_len, eos, device, &m,
                                 &err);
  if (rc) return fail(rc, std::string("ctcb_lm_create: ") + err);
  *out = new ctcb_lm{m};
  return CTCB_OK;
}

int ctcb_lm_destroy(ctcb_lm_t* lm) {
  if (!lm) return CTCB_OK;
  ctcb::lm_model_destroy(lm->m);
  delete lm;
  return CTCB_OK;
}

// Transactional: arguments are validated and the new tables built before the
// attached ones are released, so a failure leaves the previous LM in place.
int ctcb_set_lm(ctcb_t* h, const ctcb_lm_t* lm, const int32_t* token_word, double weight) {
  if (!h) return fail(CTCB_ERR_ARG, "NULL handle");
  CTCB_CUDA(cudaSetDevice(h->device));
  ctcb::LmTables fresh{};
  if (lm) {
    if (!token_word) return fail(CTCB_ERR_ARG, "token_word must not be NULL");
    if (!std::isfinite(weight)) return fail(CTCB_ERR_ARG, "lm_weight must be finite");
    if (h->beam > ctcb::kFusedMaxBeam)
      return fail(CTCB_ERR_UNSUPPORTED, "LM fusion supports beam_size <= " + std::to_string(ctcb::kFusedMaxBeam));
    if (lm->m->device != h->device) return fail(CTCB_ERR_ARG, "LM and decoder are on different devices");
    for (int c = 0; c < h->V; c++)
      if (token_word[c] < -2) return fail(CTCB_ERR_ARG, "token_word entries must be >= -2");
    const char* err = "";
    const int rc = ctcb::lm_tables_build(lm->m, token_word, h->V, weight, &fresh, &err);
    if (rc) {
      ctcb::lm_tables_free(&fresh);
      return fail(rc, std::string("ctcb_set_lm: ") + err);
    }
  }
  if (h->has_lm) {
    CTCB_CUDA(cudaDeviceSynchronize());  // decodes still reading the old tables
    ctcb::lm_tables_free(&h->lm);
    h->has_lm = 0;
  }
  if (lm) {
    h->lm = fresh;
    h->has_lm = 1;
    h->lm_weight = weight;
  }
  return CTCB_OK;
}

int ctcb_set_silence(ctcb_t* h, int sil, double sil_score) {
  if (!h) return fail(CTCB_ERR_ARG, "NULL handle");
  if (sil >= h->V) return fail(CTCB_ERR_ARG, "silence_index " + std::to_string(sil) + " out of range");
  if (sil == h->blank) return fail(CTCB_ERR_ARG, "silence_index must differ from blank_index");
  if (!std::isfinite(sil_score)) return fail(CTCB_ERR_ARG, "sil_score must be finite");
  if (sil >= 0 && sil_score != 0.0 && h->beam > ctcb::kFusedMaxBeam)
    return fail(CTCB_ERR_UNSUPPORTED, "a silence bonus supports beam_size <= " + std::to_string(ctcb::kFusedMaxBeam));
  h->sil = sil < 0 ? -1 : sil;
  h->sil_score = sil < 0 ? 0.0 : sil_score;
  return CTCB_OK;
}

// Host-buffer decode, enqueued in `nchunks` consecutive utterance ranges: per
// chunk the valid frames of each utterance go H2D on four copy streams, the
// decode stream joins them, decodes the chunk and copies its results D2H, then
// records the chunk's event.  Copies of chunk c+1 overlap the decode of c.
static int host_enqueue(ctcb_t* h, const float* lp, int64_t sb, int64_t st, const int32_t* lens, int B, int T,
                        int nchunks, void* stream, int32_t* out_tokens, int32_t* out_ts, int32_t* out_len,
                        double* out_score, int32_t* out_count, int32_t* out_status) {
  if (!h) return fail(CTCB_ERR_ARG, "NULL handle");
  if (!lp || !lens || !out_tokens || !out_len || !out_score || !out_count || !out_status)
    return fail(CTCB_ERR_ARG, "host pointers must not be NULL (out_timesteps may be)");
  h->n_chunks = 0;
  if (B <= 0) return CTCB_OK;
  if (T < 0) return fail(CTCB_ERR_ARG, "t_max must be >= 0");
  if (st < h->V || sb < (int64_t)st * (T > 0 ? T : 1))
    return fail(CTCB_ERR_ARG, "strides must describe a [batch, t_max, vocab] layout with unit vocab stride");
  if (nchunks < 1) nchunks = 1;
  if (nchunks > kMaxChunks) nchunks = kMaxChunks;
  if (nchunks > B) nchunks = B;
  CTCB_CUDA(cudaSetDevice(h->device));
  cudaStream_t s = (cudaStream_t)stream;
  const int Tp = T > 0 ? T : 1;
  const size_t V = (size_t)h->V, nb = (size_t)h->nbest;
  // device staging: dense [B, T, V] input (valid frames only are copied), lens, outputs
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t r = ctcb::align_up(o, 256); o = r + bytes; return r; };
  const size_t o_in = take((size_t)B * Tp * V * 4), o_lens = take((size_t)B * 4),
               o_tok = take((size_t)B * nb * Tp * 4), o_ts = take(out_ts ? (size_t)B * nb * Tp * 4 : 0),
               o_len = take((size_t)B * nb * 4), o_sc = take((size_t)B * nb * 8), o_cnt = take((size_t)B * 4),
               o_st = take((size_t)B * 4);
  if (h->hbuf_bytes < o) {
    if (h->hbuf) {
      CTCB_CUDA(cudaDeviceSynchronize());
      cudaFree(h->hbuf);
    }
    h->hbuf = nullptr;
    h->hbuf_bytes = 0;
    CTCB_CUDA(cudaMalloc(&h->hbuf, o));
    h->hbuf_bytes = o;
  }
  char* d = (char*)h->hbuf;
  float* din = (float*)(d + o_in);
  int32_t* dlens = (int32_t*)(d + o_lens);
  int32_t *dtok = (int32_t*)(d + o_tok), *dts = out_ts ? (int32_t*)(d + o_ts) : nullptr, *dln = (int32_t*)(d + o_len);
  double* dsc = (double*)(d + o_sc);
  int32_t *dcnt = (int32_t*)(d + o_cnt), *dst_ = (int32_t*)(d + o_st);
  if (!h->have_cstreams) {
    for (int i = 0; i < 4; i++) CTCB_CUDA(cudaStreamCreateWithFlags(&h->cstreams[i], cudaStreamNonBlocking));
    for (int i = 0; i < 5; i++) CTCB_CUDA(cudaEventCreateWithFlags(&h->cev[i], cudaEventDisableTiming));
    for (int i = 0; i < kMaxChunks; i++) CTCB_CUDA(cudaEventCreateWithFlags(&h->chunk_ev[i], cudaEventDisableTiming));
    h->have_cstreams = 1;
  }
  // page-locked input mapped into the device address space: gather it with a
  // kernel (one launch per range) instead of per-utterance DMA calls
  const float* mapped = nullptr;
  {
    cudaPointerAttributes pa{};
    if (cudaPointerGetAttributes(&pa, lp) == cudaSuccess && pa.type == cudaMemoryTypeHost && pa.devicePointer)
      mapped = (const float*)pa.devicePointer;
    cudaGetLastError();
  }
  // copies are ordered after `stream`'s prior work
  CTCB_CUDA(cudaEventRecord(h->cev[4], s));
  for (int i = 0; i < 4; i++) CTCB_CUDA(cudaStreamWaitEvent(h->cstreams[i], h->cev[4], 0));
  CTCB_CUDA(cudaMemcpyAsync(dlens, lens, (size_t)B * 4, cudaMemcpyHostToDevice, s));
  if (mapped) {
    CTCB_CUDA(cudaEventRecord(h->cev[4], s));  // lens on the device
    CTCB_CUDA(cudaStreamWaitEvent(h->cstreams[0], h->cev[4], 0));
  }
  for (int c = 0; c < nchunks; c++) {
    const int b0 = (int)((int64_t)B * c / nchunks), b1 = (int)((int64_t)B * (c + 1) / nchunks);
    if (mapped) {
      ctcb::ctcb_gather_kernel<<<2 * h->num_sms, 256, 0, h->cstreams[0]>>>(mapped, sb, st, dlens, b0, b1, T, Tp, (int)V, din);
      h->launches++;
      CTCB_CUDA(cudaGetLastError());
    }
    for (int b = b0; b < b1 && !mapped; b++) {
      int n = lens[b];
      if (n <= 0) continue;
      if (n > T) n = T;
      const float* src = lp + (size_t)b * sb;
      float* dst = din + (size_t)b * Tp * V;
      cudaStream_t cs = h->cstreams[b & 3];
      if (st == (int64_t)V)
        CTCB_CUDA(cudaMemcpyAsync(dst, src, (size_t)n * V * 4, cudaMemcpyHostToDevice, cs));
      else
        CTCB_CUDA(cudaMemcpy2DAsync(dst, V * 4, src, (size_t)st * 4, V * 4, (size_t)n, cudaMemcpyHostToDevice, cs));
    }
    for (int i = 0; i < 4; i++) {
      CTCB_CUDA(cudaEventRecord(h->cev[i], h->cstreams[i]));
      CTCB_CUDA(cudaStreamWaitEvent(s, h->cev[i], 0));
    }
    const int Bc = b1 - b0;
    const size_t r0 = (size_t)b0 * nb;
    int rc = ctcb_decode(h, din + (size_t)b0 * Tp * V, (int64_t)Tp * V, (int64_t)V, dlens + b0, Bc, T, nullptr, 0,
                         stream, dtok + r0 * Tp, dts ? dts + r0 * Tp : nullptr, dln + r0, dsc + r0, dcnt + b0, dst_ + b0);
    if (rc) return rc;
    // D2H of the chunk's results
    CTCB_CUDA(cudaMemcpyAsync(out_tokens + r0 * Tp, dtok + r0 * Tp, (size_t)Bc * nb * Tp * 4, cudaMemcpyDeviceToHost, s));
    if (out_ts)
      CTCB_CUDA(cudaMemcpyAsync(out_ts + r0 * Tp, dts + r0 * Tp, (size_t)Bc * nb * Tp * 4, cudaMemcpyDeviceToHost, s));
    CTCB_CUDA(cudaMemcpyAsync(out_len + r0, dln + r0, (size_t)Bc * nb * 4, cudaMemcpyDeviceToHost, s));
    CTCB_CUDA(cudaMemcpyAsync(out_score + r0, dsc + r0, (size_t)Bc * nb * 8, cudaMemcpyDeviceToHost, s));
    CTCB_CUDA(cudaMemcpyAsync(out_count + b0, dcnt + b0, (size_t)Bc * 4, cudaMemcpyDeviceToHost, s));
    CTCB_CUDA(cudaMemcpyAsync(out_status + b0, dst_ + b0, (size_t)Bc * 4, cudaMemcpyDeviceToHost, s));
    CTCB_CUDA(cudaEventRecord(h->chunk_ev[c], s));
    h->chunk_b0[c] = b0;
    h->chunk_b1[c] = b1;
    h->n_chunks = c + 1;
  }
  return CTCB_OK;
}

int ctcb_decode_host(ctcb_t* h, const float* lp, int64_t sb, int64_t st, const int32_t* lens, int B, int T,
                     void* stream, int32_t* out_tokens, int32_t* out_ts, int32_t* out_len, double* out_score,
                     int32_t* out_count, int32_t* out_status) {
  int rc = host_enqueue(h, lp, sb, st, lens, B, T, 1, stream, out_tokens, out_ts, out_len, out_score, out_count,
                        out_status);
  if (rc) return rc;
  CTCB_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  return CTCB_OK;
}

int ctcb_decode_host_async(ctcb_t* h, const float* lp, int64_t sb, int64_t st, const int32_t* lens, int B, int T,
                           int nchunks, void* stream, int32_t* out_tokens, int32_t* out_ts, int32_t* out_len,
                           double* out_score, int32_t* out_count, int32_t* out_status, int* chunks_out) {
  if (!chunks_out) return fail(CTCB_ERR_ARG, "chunks_out must not be NULL");
  *chunks_out = 0;
  int rc = host_enqueue(h, lp, sb, st, lens, B, T, nchunks, stream, out_tokens, out_ts, out_len, out_score,
                        out_count, out_status);
  if (h) *chunks_out = h->n_chunks;
  return rc;
}

int ctcb_decode_host_wait(ctcb_t* h, int chunk, int* b0, int* b1) {
  if (!h || !b0 || !b1) return fail(CTCB_ERR_ARG, "NULL argument");
  if (chunk < 0 || chunk >= h->n_chunks) return fail(CTCB_ERR_ARG, "chunk out of range");
  CTCB_CUDA(cudaSetDevice(h->device));
  CTCB_CUDA(cudaEventSynchronize(h->chunk_ev[chunk]));
  *b0 = h->chunk_b0[chunk];
  *b1 = h->chunk_b1[chunk];
  return CTCB_OK;
}

int ctcb_debug_frames(ctcb_t* h, const float* lp, int64_t sb, int64_t st, const int32_t* lens, int B, int T,
                      void* stream, int32_t* out_frame_map, int32_t* out_kept, int32_t* out_topk_tok,
                      float* out_topk_val, float* out_blank) {
  if (!h) return fail(CTCB_ERR_ARG, "NULL handle");
  if (!out_frame_map || !out_kept || !out_topk_tok || !out_topk_val || !out_blank)
    return fail(CTCB_ERR_ARG, "output pointers must not be NULL");
  if (B == 0) return CTCB_OK;
  CTCB_CUDA(cudaSetDevice(h->device));
  ctcb::Params P;
  WsLayout L;
  int rc = make_params(h, lp, sb, st, lens, B, T, nullptr, 0, P, L);
  if (rc) return rc;
  P.frame_map = out_frame_map;
  P.kept = out_kept;
  rc = launch_config(h, P, B, false);
  if (rc) return rc;
  size_t smem = (size_t)P.smem_per_warp;
  CTCB_CUDA(cudaFuncSetAttribute(ctcb::ctcb_debug_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  ctcb::ctcb_debug_kernel<<<B, 32, smem, (cudaStream_t)stream>>>(P, out_topk_tok, out_topk_val, out_blank);
  CTCB_CUDA(cudaGetLastError());
  return CTCB_OK;
}

int ctcb_validate(ctcb_t* h, const float* lp, int64_t sb, int64_t st, const int32_t* lens, int B, int T, int strict,
                  void* stream, int64_t* out_error) {
  if (!h || !lp || !lens || !out_error) return fail(CTCB_ERR_ARG, "NULL argument");
  if (st < h->V || sb < (int64_t)st * (T > 0 ? T : 1))
    return fail(CTCB_ERR_ARG, "strides must describe a [batch, t_max, vocab] layout with unit vocab stride");
  CTCB_CUDA(cudaSetDevice(h->device));
  cudaStream_t s = (cudaStream_t)stream;
  if (!h->ws || h->ws_bytes < 256) {
    if (h->ws) cudaFree(h->ws);
    h->ws = nullptr;
    h->ws_bytes = 0;
    CTCB_CUDA(cudaMalloc(&h->ws, 256));
    h->ws_bytes = 256;
  }
  unsigned long long* key = (unsigned long long*)h->ws;
  CTCB_CUDA(cudaMemsetAsync(key, 0xff, sizeof(unsigned long long), s));
  if (B > 0 && T > 0) {
    dim3 grid((unsigned)((T + 7) / 8), (unsigned)B);
    ctcb::ctcb_validate_kernel<<<grid, 256, 0, s>>>(lp, sb, st, lens, B, T, h->V, strict, key);
    h->launches++;
    CTCB_CUDA(cudaGetLastError());
  }
  ctcb::ctcb_validate_decode_kernel<<<1, 1, 0, s>>>(key, T, h->V, out_error);
  h->launches++;
  CTCB_CUDA(cudaGetLastError());
  return CTCB_OK;
}

}  // extern "C"
