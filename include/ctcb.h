/*
 * ctcb — B200-native (sm_100a) CTC prefix beam-search decoder: C ABI.
 *
 * The reference has no FFI for this path: its boundary is the Python call
 *   ctcforge.beam_search_decode(emissions, tokens, opts)
 *       /root/reference/pkg/src/ctcforge/decoder.py:102-135
 *   ctcforge.decode_batch(emissions, tokens, opts, workers)
 *       /root/reference/pkg/src/ctcforge/decoder.py:138-170
 * with blank skipping in ctcforge.blank_collapse (emissions.py:284-306).
 * These entry points are what a binding for that path attaches to (ctypes
 * stub in INTEGRATION.md); the Python façade `cuda_ctc_decoder` /
 * `CUCTCDecoder` (paper_2310_17864_b200/decoder.py) is built on them.
 *
 * Conventions: plain pointers and sizes; every function returns a ctcb status
 * (0 = OK).  Device pointers are CUDA device memory on the handle's device.
 * ctcb_decode only enqueues work on `stream`; outputs are valid once the
 * stream has been synchronised.  A handle is not thread-safe and is
 * single-stream: its scratch (cached workspace, host staging, debug counters)
 * is shared by all its calls, so two decodes on one handle must be ordered on
 * one stream.  Use one handle per host thread / stream.
 */
#ifndef CTCB_H
#define CTCB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ctcb_handle ctcb_t;
typedef struct ctcb_lm ctcb_lm_t;

enum {
  CTCB_OK = 0,
  CTCB_ERR_ARG = 1,          /* invalid argument (message: ctcb_last_error) */
  CTCB_ERR_CUDA = 2,         /* CUDA runtime error */
  CTCB_ERR_WORKSPACE = 3,    /* workspace too small */
  CTCB_ERR_UNSUPPORTED = 4,  /* configuration exceeds device limits */
};

/* Per-utterance status written to out_status by ctcb_decode. */
enum {
  CTCB_UTT_OK = 0,
  CTCB_UTT_EMPTY = 1,      /* len == 0: "empty emissions" (decoder.py:117-118) */
  CTCB_UTT_BAD_LEN = 2,    /* len < 0 or len > t_max */
  CTCB_UTT_BEAM_DIED = 3,  /* no finite extension survives (decoder.py:616-620); out_len[b][0] = the
                              kept-frame index where it died */
  CTCB_UTT_OVERFLOW = 4,   /* fused search (LM / silence bonus): more near-tied candidates at the
                              beam cut than the kernel's window holds; out_len[b][0] = frame */
  /* input validation (ctcb_set_validate; EmissionMatrix.__post_init__, emissions.py:128-150):
     out_len[b][0] = the first offending frame, out_count[b] = its token (-1 for NOT_NORMALIZED) */
  CTCB_UTT_NONFINITE = 5,       /* a NaN or infinite log-probability */
  CTCB_UTT_ABOVE_ZERO = 6,      /* a log-probability above MAX_LOG_PROB = 1e-4 */
  CTCB_UTT_NOT_NORMALIZED = 7,  /* |fp64 logsumexp(row)| > ROW_NORM_TOL = 1e-3 (strict mode) */
};

/* Create a decoder.  Replaces DecoderOptions (decoder.py:34-66) + the
 * TokenDictionary blank index (emissions.py:36-63) for the lexicon-free,
 * LM-free, full-vocabulary, logadd-merge configuration:
 *   vocab           V (number of emission columns)
 *   blank           blank index, 0 <= blank < V
 *   beam            beam_size, 1 <= beam <= 512
 *   nbest           n_best, 1 <= nbest <= beam
 *   skip_cutoff     drop frame t iff log_probs[t, blank] >= skip_cutoff
 *                   (+INFINITY disables skipping: blank_skip_threshold == 1.0;
 *                   see ctcb_skip_cutoff)
 *   beam_threshold  > 0; +INFINITY disables the cut (decoder.py:621-623)
 *   device          CUDA device ordinal */
int ctcb_create(int vocab, int blank, int beam, int nbest, float skip_cutoff, double beam_threshold,
                int device, ctcb_t** out);
int ctcb_destroy(ctcb_t* h);

/* Candidate merge rule (DecoderOptions.merge_mode, decoder.py:52-53, :610-613,
 * :789-791): 0 = "logadd" (default: numpy's logaddexp fold), 1 = "max"
 * (group maximum; flag variants also combined by max at finalisation). */
int ctcb_set_merge_mode(ctcb_t* h, int max_mode);

/* Token selection DecoderOptions.beam_size_token (decoder.py:440-458): per
 * frame only the K best tokens of the row, blank included, by (log-prob desc,
 * index asc) are candidates; blank groups need the blank selected, repeat
 * groups and last-token appends need the last token selected.  K <= 0 or
 * K == V: full vocabulary (the default); K > V: CTCB_ERR_ARG
 * ("beam_size_token K exceeds vocabulary size V", decoder.py:124-128). */
int ctcb_set_beam_size_token(ctcb_t* h, int K);

/* fp32 cutoff c(thr) such that, for every finite fp32 x,
 *   x >= c  <=>  exp((double)x) >= thr - 1e-12
 * i.e. ctcforge's skip rule (emissions.py:300-301, BLANK_SKIP_EPS :29).
 * thr in (0, 1]; thr == 1 returns +INFINITY (skipping disabled, :298-299). */
int ctcb_skip_cutoff(double threshold, float* cutoff);

/* Tokens kept per frame by the exact reduced search: min(2*beam, V-1). */
int ctcb_topk_size(const ctcb_t* h, int* k);

/* Device workspace needed to decode `batch` utterances padded to `t_max`. */
int ctcb_workspace_bytes(const ctcb_t* h, int batch, int t_max, size_t* bytes);

/* Decode a batch.  Replaces decode_batch (decoder.py:138-170):
 *   log_probs   device fp32, element (b, t, v) at b*stride_b + t*stride_t + v
 *   lens        device int32 [batch] valid frames per utterance
 *   workspace   device buffer of >= ctcb_workspace_bytes (NULL: the handle
 *               allocates and caches one)
 *   stream      cudaStream_t (NULL: legacy default stream)
 * Outputs (device):
 *   out_tokens     int32 [batch, nbest, t_max] token ids of each hypothesis
 *   out_timesteps  int32 [batch, nbest, t_max] original frame of each token
 *                  (Hypothesis.timesteps, decoder.py:69-83), or NULL
 *   out_len        int32 [batch, nbest] tokens per hypothesis
 *   out_score      float64 [batch, nbest] hypothesis score (logadd of the
 *                  prefix's blank / non-blank variants, decoder.py:789-791)
 *   out_count      int32 [batch] hypotheses returned (<= nbest)
 *   out_status     int32 [batch] CTCB_UTT_* per utterance */
int ctcb_decode(ctcb_t* h, const float* log_probs, int64_t stride_b, int64_t stride_t, const int32_t* lens,
                int batch, int t_max, void* workspace, size_t workspace_bytes, void* stream,
                int32_t* out_tokens, int32_t* out_timesteps, int32_t* out_len, double* out_score,
                int32_t* out_count, int32_t* out_status);

/* Decode from HOST memory (the e2e path a host-side binding uses): copies the
 * valid frames of each utterance host->device (pinned memory makes the copies
 * asynchronous DMA), decodes, copies the results back and synchronises
 * `stream`.  Same layouts as ctcb_decode with host pointers throughout;
 * lens are read on the host.  Device staging is cached in the handle. */
int ctcb_decode_host(ctcb_t* h, const float* log_probs, int64_t stride_b, int64_t stride_t, const int32_t* lens,
                     int batch, int t_max, void* stream, int32_t* out_tokens, int32_t* out_timesteps,
                     int32_t* out_len, double* out_score, int32_t* out_count, int32_t* out_status);

/* Chunked, asynchronous form of ctcb_decode_host for pipelined callers:
 * splits the batch into `nchunks` (<= 64) consecutive utterance ranges and
 * enqueues, per range, the H2D copies of its valid frames, its decode and the
 * D2H of its results into the host output buffers (pinned memory keeps the
 * copies asynchronous), then returns without synchronising; *chunks_out is
 * the number of ranges.  The H2D copies of range c+1 overlap the decode of c.
 * ctcb_decode_host_wait blocks until range `chunk` is on the host and reports
 * it as [*b0, *b1).  Host buffers must stay valid until the last wait. */
int ctcb_decode_host_async(ctcb_t* h, const float* log_probs, int64_t stride_b, int64_t stride_t,
                           const int32_t* lens, int batch, int t_max, int nchunks, void* stream,
                           int32_t* out_tokens, int32_t* out_timesteps, int32_t* out_len, double* out_score,
                           int32_t* out_count, int32_t* out_status, int* chunks_out);
int ctcb_decode_host_wait(ctcb_t* h, int chunk, int* b0, int* b1);

/* Debug / minimum slice: blank-skip compaction and per-frame top-k only.
 * Replaces blank_collapse (emissions.py:284-306) and the token selection of
 * _BeamSearch._step (decoder.py:431-460, :440):
 *   out_frame_map  int32 [batch, t_max]   kept original frames (first out_kept[b])
 *   out_kept       int32 [batch]
 *   out_topk_tok   int32 [batch, t_max, k] best non-blank tokens of each kept
 *                  frame by (log-prob desc, index asc), k = ctcb_topk_size
 *   out_topk_val   float [batch, t_max, k] their log-probs
 *   out_blank      float [batch, t_max]   the blank log-prob of each kept frame */
int ctcb_debug_frames(ctcb_t* h, const float* log_probs, int64_t stride_b, int64_t stride_t,
                      const int32_t* lens, int batch, int t_max, void* stream, int32_t* out_frame_map,
                      int32_t* out_kept, int32_t* out_topk_tok, float* out_topk_val, float* out_blank);

/* Input validation fused into every decode (default mode 1), replacing
 * EmissionMatrix(strict=True).__post_init__ (emissions.py:128-150) that
 * ctcforge runs on each utterance before decoding: mode 0 off, 1 strict,
 * 2 without the normalisation check (strict=False).  The decode kernels screen
 * each row as they stage it; rows they do not stage (blank-skipped frames,
 * frames after a dead beam) are checked by a follow-up kernel.  An invalid
 * utterance's out_status is CTCB_UTT_NONFINITE / _ABOVE_ZERO / _NOT_NORMALIZED
 * for its first offender in the reference's order, overriding the decode's. */
int ctcb_set_validate(ctcb_t* h, int mode);

/* Validation pass mirroring EmissionMatrix(strict=True) (emissions.py:128-150):
 * first offending (b, t, v) of: non-finite value (code 1), value > 1e-4
 * (code 2), |logsumexp(row)| > 1e-3 (code 3, v = -1).  out_error: device
 * int64 [4] = {code, b, t, v}, code 0 if clean. Frames t >= lens[b] are ignored. */
int ctcb_validate(ctcb_t* h, const float* log_probs, int64_t stride_b, int64_t stride_t, const int32_t* lens,
                  int batch, int t_max, int strict, void* stream, int64_t* out_error);

/* Diagnostics of the last ctcb_decode on this handle (synchronising read):
 * {key ties resolved exactly, exact fp64 score ties, token-sequence
 *  materialisations, trellis steps walked by them, radix top-k fallbacks, 0,
 *  truncated-key top-k fixups, one-shot selection fallbacks to the k-way merge}. */
int ctcb_debug_counters(ctcb_t* h, uint64_t* out8);

/* Kernel timing for measurement: while enabled, every ctcb_decode records a
 * CUDA event pair around its beam-search kernel on the decode stream (up to 64
 * launches; enabling resets the list).  ctcb_kernel_time synchronises on the
 * last pair and returns the summed kernel time, the number of timed launches
 * and the name of the last kernel launched (static storage). */
int ctcb_kernel_timing(ctcb_t* h, int enable);
int ctcb_kernel_time(ctcb_t* h, double* total_ms, int* launches, const char** kernel);

/* Number of CUDA kernels this handle has launched so far (decode, gather,
 * validation; host-side counter, no synchronisation).  bench.py reads it
 * around the timed region for its gpu_launches field. */
int ctcb_launch_count(ctcb_t* h, uint64_t* out);

/* ---- CTC forced alignment (ctcforge align.py:46-123) ----------------------
 * Viterbi over each utterance's blank-interleaved targets, one warp per
 * utterance, fp64 path scores with the reference's tie-breaking (stay over
 * advance-1 over advance-2; the final blank over the final token):
 *   log_probs        device fp32 [batch, t_max, vocab] (strides as ctcb_decode)
 *   lens             device int32 [batch] frames per utterance
 *   targets          device int32, all utterances' target tokens concatenated
 *   target_offsets   device int32 [batch + 1] (utterance b: [off[b], off[b+1]))
 *   s_max            >= 2 * max targets + 1
 *   workspace        device >= ctcb_align_workspace_bytes(batch, t_max, s_max)
 * Outputs (device): out_labels int32 [batch, t_max] token per frame (blank
 * allowed), out_scores fp32 [batch, t_max] its log-prob, out_status int32
 * [batch] CTCB_ALIGN_*, and (optional, NULL to skip) the token spans:
 * out_span_start / out_span_end int32 in the targets' layout, target j of
 * utterance b occupies frames [start, end) (align.py:126-143's spans, one per
 * target).  Enqueued on `stream` (on the current device). */
enum {
  CTCB_ALIGN_OK = 0,
  CTCB_ALIGN_EMPTY_TARGETS = 1,  /* "targets must be non-empty" (align.py:62-63) */
  CTCB_ALIGN_BLANK_TARGET = 2,   /* "targets must not contain the blank token" (:64-66) */
  CTCB_ALIGN_RANGE = 3,          /* "target token t out of range [0, V)" (:67-68) */
  CTCB_ALIGN_INFEASIBLE = 4,     /* T < L + adjacent repeats (:69-75) */
  CTCB_ALIGN_NO_PATH = 5,        /* "no feasible alignment path" (:108-110) */
  CTCB_ALIGN_BAD_LEN = 6,        /* length outside [0, t_max] or targets beyond s_max */
};
int ctcb_align_workspace_bytes(int batch, int t_max, int s_max, size_t* bytes);
int ctcb_align(const float* log_probs, int64_t stride_b, int64_t stride_t, const int32_t* lens,
               const int32_t* targets, const int32_t* target_offsets, int batch, int t_max, int vocab, int blank,
               int s_max, void* workspace, size_t workspace_bytes, void* stream, int32_t* out_labels,
               float* out_scores, int32_t* out_status, int32_t* out_span_start, int32_t* out_span_end);

/* ---- Token-level LM fusion ---------------------------
 * Replaces NGramLM + parse_arpa (lm.py:35-226) on the device and the
 * lexicon-free fusion of _BeamSearch (decoder.py:178-259, :467-486, :753-817).
 *
 * ctcb_lm_create uploads a flattened backoff model: n-gram i has
 * words[i * order .. + lengths[i]) (word ids >= 0), natural-log logprob[i] and
 * backoff[i]; a repeated tuple keeps its last row.  `start` (start_len <=
 * order - 1 words) is the start context (lm.py:229-233: "<s>" shrunk to a known
 * context, or empty); `eos` the word id scored at the end ("</s>", else
 * "<unk>", else -1 for the OOV penalty).  order <= 8. */
int ctcb_lm_create(int order, int64_t n_ngrams, const int32_t* words, const int32_t* lengths, const double* logprob,
                   const double* backoff, const int32_t* start, int start_len, int eos, int device,
                   ctcb_lm_t** out);
int ctcb_lm_destroy(ctcb_lm_t* lm);
/* Attach a model to a decoder (NULL detaches): builds the dense context x
 * token score / successor tables on the device.  token_word[c] (host, V
 * entries): the LM word id of token c (its string, or "<unk>"), -1 when the
 * string is out of vocabulary and the model has no "<unk>" (fixed penalty
 * -20, context reset: lm.py:236-238), -2 for blank and the silence token
 * (identity: no LM score, context kept).  weight: lm_weight.  beam <= 128. */
int ctcb_set_lm(ctcb_t* h, const ctcb_lm_t* lm, const int32_t* token_word, double weight);
/* Silence token (-1: none) and its per-emission bonus sil_score
 * (decoder.py:485-486); a non-zero bonus selects the fused search (beam <= 128). */
int ctcb_set_silence(ctcb_t* h, int silence_index, double sil_score);
/* ctcb_decode plus out_lm: float64 [batch, nbest] LM total of each hypothesis
 * (Hypothesis.lm_score, finish score included; decoder.py:770-777), or NULL.
 * Scores include lm_weight * LM and the silence bonuses. */
int ctcb_decode_lm(ctcb_t* h, const float* log_probs, int64_t stride_b, int64_t stride_t, const int32_t* lens,
                   int batch, int t_max, void* workspace, size_t workspace_bytes, void* stream,
                   int32_t* out_tokens, int32_t* out_timesteps, int32_t* out_len, double* out_score,
                   double* out_lm, int32_t* out_count, int32_t* out_status);

const char* ctcb_status_string(int status);
/* Message of the last error on this host thread. */
const char* ctcb_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* CTCB_H */
