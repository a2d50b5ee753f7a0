"""Drop-in CUDA CTC decoder façade: ``cuda_ctc_decoder`` / ``CUCTCDecoder``.

Signature of the north-star API (TorchAudio's ``cuda_ctc_decoder``), semantics
of the reference CPU decoder (ctcforge):

    decoder = cuda_ctc_decoder(tokens, nbest=1, beam_size=10, blank_skip_threshold=0.95)
    hyps = decoder(log_probs, encoder_out_lens)   # List[List[CUCTCHypothesis]]

For every utterance b the result equals the reference call

    beam_search_decode(EmissionMatrix(log_probs[b, :len_b] as float64),
                       TokenDictionary(tokens, blank_index=0),
                       DecoderOptions(beam_size, n_best=nbest,
                                      blank_skip_threshold=blank_skip_threshold,
                                      beam_size_token=None, beam_threshold=50.0,
                                      merge_mode="logadd"))

(decoder.py:102-135) mapped to ``CUCTCHypothesis(tokens, words=[tokens[i]...],
score)``.  Errors follow ctcforge: option errors raise ``ValueError`` with
DecoderOptions' messages (decoder.py:54-66), token-dictionary errors with
TokenDictionary's (emissions.py:49-58), a zero-length utterance raises
``ValueError("utterance b: empty emissions")`` (decoder.py:117-118, :157).

All compute runs in libctcb.so (sm_100a kernels); this module only checks
arguments, allocates through PyTorch's caching allocator and converts results.
"""

from __future__ import annotations

import contextlib
import ctypes
import gc
from typing import List, NamedTuple, Optional, Union

import numpy as np
import torch

from . import _lib

__all__ = ["CUCTCHypothesis", "CUCTCDecoder", "cuda_ctc_decoder", "skip_cutoff", "DecodeOutput"]

_DEFAULT_BLANK_SKIP_THRESHOLD = 0.95
BLANK_SKIP_EPS = 1e-12  # emissions.py:29
MAX_BEAM = 512


class CUCTCHypothesis(NamedTuple):
    """One n-best entry (TorchAudio's CUCTCHypothesis fields)."""

    tokens: List[int]
    words: List[str]
    score: float


class DecodeOutput(NamedTuple):
    """Raw device outputs of one decode call (see include/ctcb.h)."""

    tokens: torch.Tensor      # int32 [B, nbest, T]
    timesteps: Optional[torch.Tensor]  # int32 [B, nbest, T] or None
    lengths: torch.Tensor     # int32 [B, nbest]
    scores: torch.Tensor      # float64 [B, nbest]
    counts: torch.Tensor      # int32 [B]
    status: torch.Tensor      # int32 [B]
    lm: Optional[torch.Tensor] = None  # float64 [B, nbest] LM totals (decoder with an LM attached)
    inputs: Optional[torch.Tensor] = None  # the decoded log_prob (validation error messages)


def validation_message(code: int, row, t: int, v: int) -> str:
    """EmissionMatrix.__post_init__'s message (emissions.py:133-150) for check
    ``code`` (1 non-finite, 2 above 0, 3 not normalized) at frame t, token v;
    ``row`` is frame t's log-probs (values for the message)."""
    if code == 1:
        return f"non-finite log-probability at frame {t}, token {v}"
    x = torch.as_tensor(row).double().cpu() if row is not None else None
    if code == 2:
        return f"log-probability above 0 at frame {t}, token {v}: {float(x[v]) if x is not None else float('nan'):.6g}"
    norm = float(torch.logsumexp(x, 0)) if x is not None else float("nan")
    return (f"frame {t} is not normalized: log-sum-exp = {norm:.6g} (tolerance 0.001); "
            "pass strict=False to skip this check")


def _read_vocab(path: str) -> list[str]:
    # first whitespace-separated field of each line (TorchAudio's _get_vocab_list)
    vocab = []
    with open(path, "r", encoding="utf-8") as fh:
        for line in fh:
            fields = line.strip().split()
            vocab.append(fields[0] if fields else "")
    return vocab


def _check_tokens(tokens: list[str]) -> None:
    # TokenDictionary invariants, emissions.py:49-58
    if not tokens:
        raise ValueError("token dictionary is empty")
    if any(not t for t in tokens):
        raise ValueError("token strings must be non-empty")
    if len(set(tokens)) != len(tokens):
        raise ValueError("token strings must be unique")


def skip_cutoff(threshold: float) -> float:
    """fp32 cutoff c with ``x >= c  <=>  exp(float64(x)) >= threshold - 1e-12``
    for every finite fp32 x: ctcforge's blank-skip rule (emissions.py:300-301)
    evaluated with numpy's exp exactly as the reference does.  +inf for
    threshold == 1.0 (skipping disabled, emissions.py:298-299)."""
    if not 0.0 < threshold <= 1.0:
        raise ValueError("blank_skip_threshold must be in (0, 1]")
    if threshold == 1.0:
        return float("inf")
    target = threshold - BLANK_SKIP_EPS
    if not target > 0.0:
        return float("-inf")

    def drop(x: np.float32) -> bool:
        return bool(np.exp(np.array([x], dtype=np.float32).astype(np.float64))[0] >= target)

    c = np.float32(np.log(target))
    down = np.float32(-np.inf)
    while drop(np.nextafter(c, down)):
        c = np.nextafter(c, down)
    while not drop(c):
        c = np.nextafter(c, np.float32(np.inf))
    return float(c)


class CUCTCDecoder:
    """CUDA CTC prefix beam-search decoder (build with :func:`cuda_ctc_decoder`).

    One decoder = one C handle = one stream: its scratch buffers are reused
    by every call, so calls are enqueued on ``cuda_stream`` (or the current
    stream at construction) and must not be issued concurrently from several
    threads or streams; use one decoder per stream (see MultiDeviceDecoder)."""

    def __init__(
        self,
        vocab_list: List[str],
        blank_id: int = 0,
        beam_size: int = 10,
        nbest: int = 1,
        blank_skip_threshold: float = _DEFAULT_BLANK_SKIP_THRESHOLD,
        cuda_stream: Optional[torch.cuda.Stream] = None,
        beam_threshold: float = 50.0,
        validate: bool = True,
        device: Optional[Union[int, torch.device]] = None,
    ):
        vocab_list = list(vocab_list)
        _check_tokens(vocab_list)
        if not 0 <= blank_id < len(vocab_list):
            raise ValueError(f"blank_index {blank_id} out of range")
        # DecoderOptions.__post_init__, decoder.py:54-66
        if beam_size < 1:
            raise ValueError("beam_size must be >= 1")
        if not beam_threshold > 0:
            raise ValueError("beam_threshold must be positive")
        if not 0.0 < blank_skip_threshold <= 1.0:
            raise ValueError("blank_skip_threshold must be in (0, 1]")
        if not 1 <= nbest <= beam_size:
            raise ValueError("n_best must be in [1, beam_size]")
        if beam_size > MAX_BEAM:
            raise ValueError(f"beam_size must be <= {MAX_BEAM} for the CUDA decoder")
        if cuda_stream is not None and not isinstance(cuda_stream, torch.cuda.Stream):
            raise TypeError("cuda_stream must be torch.cuda.Stream")
        self.vocab_list = vocab_list
        self.beam_size_token: Optional[int] = None  # full vocabulary (set_beam_size_token)
        self._vocab_np = np.array(vocab_list, dtype=object)
        self.blank_id = blank_id
        self.beam_size = beam_size
        self.nbest = nbest
        self.blank_skip_threshold = blank_skip_threshold
        self.beam_threshold = float(beam_threshold)
        self.validate = validate
        self.cuda_stream = cuda_stream
        self.cutoff = skip_cutoff(blank_skip_threshold)
        if device is None:
            device = torch.cuda.current_device()
        self.device = torch.device("cuda", device if isinstance(device, int) else device.index or 0)
        lib = _lib.load()
        h = ctypes.c_void_p()
        _lib.check(lib.ctcb_create(len(vocab_list), blank_id, beam_size, nbest, ctypes.c_float(self.cutoff),
                                   self.beam_threshold, self.device.index, ctypes.byref(h)), "ctcb_create")
        self._h = h
        self.set_validate(validate)
        k = ctypes.c_int()
        _lib.check(lib.ctcb_topk_size(h, ctypes.byref(k)), "ctcb_topk_size")
        self.topk = k.value
        self._ws = None
        self._lm = None          # ctcb_lm_t of the attached model (set_lm)
        self.lm_weight = 0.0
        self.silence_index: Optional[int] = None
        self.sil_score = 0.0

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib._lib is not None:
            _lib._lib.ctcb_destroy(h)
            self._h = None
        m = getattr(self, "_lm", None)
        if m is not None and m.value and _lib._lib is not None:
            _lib._lib.ctcb_lm_destroy(m)
            self._lm = None

    # ------------------------------------------------------------------ helpers
    def _stream(self):
        s = self.cuda_stream if self.cuda_stream is not None else torch.cuda.current_stream(self.device)
        return ctypes.c_void_p(s.cuda_stream)

    def _on_stream(self):
        # with an explicit cuda_stream, output allocation/initialisation, the
        # launch and the result copies are all ordered on that stream
        return torch.cuda.stream(self.cuda_stream) if self.cuda_stream is not None else contextlib.nullcontext()

    def _check_inputs(self, log_prob: torch.Tensor, lens: torch.Tensor):
        if not isinstance(log_prob, torch.Tensor) or log_prob.dim() != 3:
            raise ValueError("log_prob must be a 3-D tensor [batch, frames, tokens]")
        if log_prob.dtype != torch.float32:
            raise ValueError(f"log_prob must be float32, got {log_prob.dtype}")
        if not log_prob.is_cuda:
            raise ValueError("log_prob must be a CUDA tensor (CPU tensors: use __call__ or decode_host)")
        B, T, V = log_prob.shape
        if V != len(self.vocab_list):
            raise ValueError(f"emissions have {V} columns but the token dictionary has "
                             f"{len(self.vocab_list)} tokens")  # decoder.py:119-123
        if not isinstance(lens, torch.Tensor) or lens.dim() != 1 or lens.shape[0] != B:
            raise ValueError("encoder_out_lens must be a 1-D tensor with one length per utterance")
        if log_prob.device != self.device:
            raise ValueError(f"log_prob is on {log_prob.device}, decoder on {self.device}")
        if log_prob.stride(2) != 1 and V > 1:
            log_prob = log_prob.contiguous()
        # strides of size-1 dims are arbitrary (numpy's [None] gives 0): use the dense value
        st = log_prob.stride(1) if T > 1 else V
        sb = log_prob.stride(0) if B > 1 else st * max(T, 1)
        if st < V or sb < st * max(T, 1):
            log_prob = log_prob.contiguous()
            st, sb = V, V * max(T, 1)
        lens = lens.to(device=self.device, dtype=torch.int32).contiguous()
        self._strides = (sb, st)
        return log_prob, lens

    def _workspace(self, B: int, T: int) -> torch.Tensor:
        lib = _lib.load()
        n = ctypes.c_size_t()
        _lib.check(lib.ctcb_workspace_bytes(self._h, B, T, ctypes.byref(n)), "ctcb_workspace_bytes")
        if self._ws is None or self._ws.numel() < n.value:
            self._ws = torch.empty(max(n.value, 1), dtype=torch.uint8, device=self.device)
        return self._ws

    def validate_inputs(self, log_prob: torch.Tensor, encoder_out_lens: torch.Tensor, strict: bool = True) -> None:
        """Standalone validation pass (ctcb_validate) without decoding: raise
        the reference's ValueError for the first invalid utterance.  Decodes
        validate on their own (set_validate); this is the explicit check."""
        log_prob, lens = self._check_inputs(log_prob, encoder_out_lens)
        lib = _lib.load()
        B, T, _ = log_prob.shape
        err = torch.empty(4, dtype=torch.int64, device=self.device)
        with self._on_stream():
            _lib.check(lib.ctcb_validate(self._h, ctypes.c_void_p(log_prob.data_ptr()), self._strides[0],
                                         self._strides[1], ctypes.c_void_p(lens.data_ptr()), B, T, int(strict),
                                         self._stream(), ctypes.c_void_p(err.data_ptr())), "ctcb_validate")
            code, b, t, v = err.cpu().tolist()
        if code:
            raise ValueError(f"utterance {b}: " + validation_message(code, log_prob[b, t], t, v))

    # ------------------------------------------------------------------ API
    def decode(self, log_prob: torch.Tensor, encoder_out_lens: torch.Tensor, timesteps: bool = False,
               offset: int = 0) -> DecodeOutput:
        """Enqueue a decode on the decoder's stream and return device tensors
        (no synchronisation).  ``offset`` shifts the batch indices in error
        messages (a range of a larger batch)."""
        with self._on_stream():
            return self._decode(log_prob, encoder_out_lens, timesteps, offset)

    def _decode(self, log_prob, encoder_out_lens, timesteps: bool, offset: int) -> DecodeOutput:
        log_prob, lens = self._check_inputs(log_prob, encoder_out_lens)
        lib = _lib.load()
        B, T, _ = log_prob.shape
        dev = self.device
        nb = self.nbest
        out_tok = torch.empty((B, nb, max(T, 1)), dtype=torch.int32, device=dev)
        out_ts = torch.empty((B, nb, max(T, 1)), dtype=torch.int32, device=dev) if timesteps else None
        out_len = torch.zeros((B, nb), dtype=torch.int32, device=dev)
        out_score = torch.zeros((B, nb), dtype=torch.float64, device=dev)
        out_count = torch.zeros(B, dtype=torch.int32, device=dev)
        out_status = torch.full((B,), -1, dtype=torch.int32, device=dev)  # -1: not processed
        ws = self._workspace(B, T)
        vp = ctypes.c_void_p
        if self._lm is not None:
            out_lm = torch.zeros((B, nb), dtype=torch.float64, device=dev)
            _lib.check(lib.ctcb_decode_lm(
                self._h, vp(log_prob.data_ptr()), self._strides[0], self._strides[1], vp(lens.data_ptr()), B, T,
                vp(ws.data_ptr()), ws.numel(), self._stream(), vp(out_tok.data_ptr()),
                vp(out_ts.data_ptr()) if out_ts is not None else None, vp(out_len.data_ptr()),
                vp(out_score.data_ptr()), vp(out_lm.data_ptr()), vp(out_count.data_ptr()),
                vp(out_status.data_ptr())), "ctcb_decode_lm")
            return DecodeOutput(out_tok, out_ts, out_len, out_score, out_count, out_status, out_lm, log_prob)
        _lib.check(lib.ctcb_decode(
            self._h, vp(log_prob.data_ptr()), self._strides[0], self._strides[1], vp(lens.data_ptr()), B, T,
            vp(ws.data_ptr()), ws.numel(), self._stream(), vp(out_tok.data_ptr()),
            vp(out_ts.data_ptr()) if out_ts is not None else None, vp(out_len.data_ptr()),
            vp(out_score.data_ptr()), vp(out_count.data_ptr()), vp(out_status.data_ptr())), "ctcb_decode")
        return DecodeOutput(out_tok, out_ts, out_len, out_score, out_count, out_status, None, log_prob)

    def to_host(self, out: DecodeOutput, offset: int = 0):
        """Synchronise and copy results to the host; raise the reference's
        errors for failed utterances (batch indices shifted by ``offset``).
        Returns numpy arrays (tokens [B, nbest, Lmax], timesteps or None,
        lengths, scores, counts)."""
        with self._on_stream():
            return self._to_host(out, offset)

    def _to_host(self, out: DecodeOutput, offset: int):
        status = out.status.cpu().numpy()
        counts = out.counts.cpu().numpy()
        lengths = out.lengths.cpu().numpy()
        self._raise_status(status, out.tokens.shape[2], lengths, offset, counts, out.inputs)
        scores = out.scores.cpu().numpy()
        lmax = int(lengths.max()) if lengths.size else 0
        tokens = out.tokens[:, :, :lmax].cpu().numpy()
        ts = out.timesteps[:, :, :lmax].cpu().numpy() if out.timesteps is not None else None
        return tokens, ts, lengths, scores, counts

    def decode_host(self, log_prob: torch.Tensor, encoder_out_lens, timesteps: bool = False):
        """Host-buffer path through ``ctcb_decode_host``: ``log_prob`` a CPU
        float32 [B, T, V] tensor (pin it for asynchronous DMA); only each
        utterance's valid frames cross PCIe.  Returns numpy (tokens, timesteps
        or None, lengths, scores, counts) like :meth:`to_host`."""
        if not isinstance(log_prob, torch.Tensor) or log_prob.dim() != 3 or log_prob.is_cuda:
            raise ValueError("decode_host expects a 3-D CPU tensor [batch, frames, tokens]")
        if log_prob.dtype != torch.float32:
            raise ValueError(f"log_prob must be float32, got {log_prob.dtype}")
        B, T, V = log_prob.shape
        if V != len(self.vocab_list):
            raise ValueError(f"emissions have {V} columns but the token dictionary has "
                             f"{len(self.vocab_list)} tokens")
        if log_prob.stride(2) != 1:
            log_prob = log_prob.contiguous()
        lens = np.ascontiguousarray(np.asarray(encoder_out_lens.cpu() if isinstance(encoder_out_lens, torch.Tensor)
                                               else encoder_out_lens, dtype=np.int32))
        if lens.shape != (B,):
            raise ValueError("encoder_out_lens must be a 1-D tensor with one length per utterance")
        st = log_prob.stride(1) if T > 1 else V
        sb = log_prob.stride(0) if B > 1 else st * max(T, 1)
        nb, Tp = self.nbest, max(T, 1)
        tok = np.empty((B, nb, Tp), dtype=np.int32)
        ts = np.empty((B, nb, Tp), dtype=np.int32) if timesteps else None
        ln = np.zeros((B, nb), dtype=np.int32)
        sc = np.zeros((B, nb), dtype=np.float64)
        cnt = np.zeros(B, dtype=np.int32)
        status = np.full(B, -1, dtype=np.int32)
        vp = ctypes.c_void_p
        lib = _lib.load()
        _lib.check(lib.ctcb_decode_host(self._h, vp(log_prob.data_ptr()), sb, st, vp(lens.ctypes.data), B, T,
                                        self._stream(), vp(tok.ctypes.data), vp(ts.ctypes.data) if ts is not None else None,
                                        vp(ln.ctypes.data), vp(sc.ctypes.data), vp(cnt.ctypes.data),
                                        vp(status.ctypes.data)), "ctcb_decode_host")
        self._raise_status(status, T, ln, 0, cnt, log_prob)
        lmax = int(ln.max()) if ln.size else 0
        return tok[:, :, :lmax], (ts[:, :, :lmax] if ts is not None else None), ln, sc, cnt

    def _pinned_outputs(self, B: int, Tp: int):
        """Page-locked host output buffers (cached per shape) so the D2H copies of
        the chunked host path are asynchronous DMA."""
        key = (B, Tp)
        if getattr(self, "_pin_key", None) != key:
            nb = self.nbest
            mk = lambda shape, dt: torch.empty(shape, dtype=dt, pin_memory=True)
            self._pin = (mk((B, nb, Tp), torch.int32), mk((B, nb), torch.int32), mk((B, nb), torch.float64),
                         mk((B,), torch.int32), mk((B,), torch.int32))
            self._pin_key = key
        return [t.numpy() for t in self._pin]

    def _decode_host_chunks(self, log_prob: torch.Tensor, encoder_out_lens, chunks: int, offset: int = 0):
        """Pipelined host path (``ctcb_decode_host_async``): yields
        (b0, b1, tokens, lengths, scores, counts) per utterance range as soon as
        that range's results are on the host, while later ranges are still
        being copied and decoded."""
        if not isinstance(log_prob, torch.Tensor) or log_prob.dim() != 3 or log_prob.is_cuda:
            raise ValueError("expected a 3-D CPU tensor [batch, frames, tokens]")
        if log_prob.dtype != torch.float32:
            raise ValueError(f"log_prob must be float32, got {log_prob.dtype}")
        B, T, V = log_prob.shape
        if V != len(self.vocab_list):
            raise ValueError(f"emissions have {V} columns but the token dictionary has "
                             f"{len(self.vocab_list)} tokens")
        if log_prob.stride(2) != 1:
            log_prob = log_prob.contiguous()
        lens = np.ascontiguousarray(np.asarray(encoder_out_lens.cpu() if isinstance(encoder_out_lens, torch.Tensor)
                                               else encoder_out_lens, dtype=np.int32))
        if lens.shape != (B,):
            raise ValueError("encoder_out_lens must be a 1-D tensor with one length per utterance")
        st = log_prob.stride(1) if T > 1 else V
        sb = log_prob.stride(0) if B > 1 else st * max(T, 1)
        Tp = max(T, 1)
        tok, ln, sc, cnt, status = self._pinned_outputs(B, Tp)
        status.fill(-1)
        vp = ctypes.c_void_p
        lib = _lib.load()
        n = ctypes.c_int()
        _lib.check(lib.ctcb_decode_host_async(self._h, vp(log_prob.data_ptr()), sb, st, vp(lens.ctypes.data), B, T,
                                              chunks, self._stream(), vp(tok.ctypes.data), None, vp(ln.ctypes.data),
                                              vp(sc.ctypes.data), vp(cnt.ctypes.data), vp(status.ctypes.data),
                                              ctypes.byref(n)), "ctcb_decode_host_async")
        b0, b1 = ctypes.c_int(), ctypes.c_int()
        for c in range(n.value):
            _lib.check(lib.ctcb_decode_host_wait(self._h, c, ctypes.byref(b0), ctypes.byref(b1)),
                       "ctcb_decode_host_wait")
            lo, hi = b0.value, b1.value
            if (status[lo:hi] != _lib.UTT_OK).any():
                _lib.check(lib.ctcb_decode_host_wait(self._h, n.value - 1, ctypes.byref(b0), ctypes.byref(b1)),
                           "ctcb_decode_host_wait")  # drain before raising
                err = status.copy()
                err[:lo] = _lib.UTT_OK
                self._raise_status(err, T, ln, offset, cnt, log_prob)
            yield lo, hi, tok[lo:hi], ln[lo:hi], sc[lo:hi], cnt[lo:hi]

    def _raise_status(self, status: np.ndarray, T: int, lengths=None, offset: int = 0, counts=None,
                      inputs=None) -> None:
        # ``offset``: batch index of status[0] in the caller's batch (multi-device ranges)
        if (status < 0).any():
            raise _lib.CtcbError(f"ctcb_decode left {(status < 0).sum()} utterance(s) unprocessed (kernel did not run)")
        bad = np.flatnonzero(status != _lib.UTT_OK)
        if bad.size:
            b = int(bad[0])
            u = b + offset
            if status[b] == _lib.UTT_EMPTY:
                raise ValueError(f"utterance {u}: empty emissions")
            if status[b] in (_lib.UTT_NONFINITE, _lib.UTT_ABOVE_ZERO, _lib.UTT_NOT_NORMALIZED):
                t, v = int(np.asarray(lengths)[b, 0]), int(np.asarray(counts)[b])
                row = inputs[b, t] if inputs is not None else None
                raise ValueError(f"utterance {u}: " + validation_message(int(status[b]) - 4, row, t, v))
            if status[b] == _lib.UTT_OVERFLOW:
                t = int(np.asarray(lengths)[b, 0]) if lengths is not None else "?"
                raise _lib.CtcbError(f"utterance {u}: frame {t}: more near-tied candidates at the beam cut than "
                                     "the fused search window holds")
            if status[b] == _lib.UTT_BEAM_DIED:
                # decoder.py:616-620; the kernel leaves the kept-frame index in lengths[b, 0]
                t = int(np.asarray(lengths)[b, 0]) if lengths is not None else "?"
                K = self.beam_size_token or len(self.vocab_list)
                raise ValueError(f"utterance {u}: beam died at frame {t}: no extension survives "
                                 f"(beam_size_token={K} may be too small)")
            raise ValueError(f"utterance {u}: length out of range [1, {T}]")

    def __call__(self, log_prob: torch.Tensor, encoder_out_lens: torch.Tensor) -> List[List[CUCTCHypothesis]]:
        """Decode a batch: ``log_prob`` float32 [B, T, V] (log-softmax output),
        ``encoder_out_lens`` [B] valid frames per utterance.  CUDA tensors are
        decoded in place (TorchAudio's contract); CPU tensors go through the
        host-buffer path (``ctcb_decode_host``).  Returns the sorted n-best per
        utterance (fewer than ``nbest`` when fewer distinct prefixes survive,
        decoder.py:801)."""
        if isinstance(log_prob, torch.Tensor) and not log_prob.is_cuda:
            # pipelined: hypotheses of range c are built while c+1.. are copied/decoded
            B = log_prob.shape[0] if log_prob.dim() == 3 else 0
            chunks = max(1, min(16, B // 256))
            result = []
            for _, _, tokens, lengths, scores, counts in self._decode_host_chunks(log_prob, encoder_out_lens, chunks):
                result.extend(self._hypotheses(tokens, lengths, scores, counts))
            return result
        else:
            out = self.decode(log_prob, encoder_out_lens)
            tokens, _, lengths, scores, counts = self.to_host(out)
        return self._hypotheses(tokens, lengths, scores, counts)

    def _hypotheses(self, tokens, lengths, scores, counts) -> List[List[CUCTCHypothesis]]:
        # one tolist() per hypothesis; words through an object-array gather.
        # The cyclic garbage collector is paused while the (acyclic) result is
        # built: its generation scans over the growing list otherwise double
        # the cost for a few thousand utterances.
        vocab = self._vocab_np
        result = []
        paused = gc.isenabled()
        if paused:
            gc.disable()
        try:
            for b in range(tokens.shape[0]):
                hyps = []
                for j in range(int(counts[b])):
                    t = tokens[b, j, : lengths[b, j]]
                    hyps.append(CUCTCHypothesis(tokens=t.tolist(), words=vocab[t].tolist(), score=float(scores[b, j])))
                result.append(hyps)
        finally:
            if paused:
                gc.enable()
        return result

    def set_merge_mode(self, mode: str) -> None:
        """``"logadd"`` (default) or ``"max"``: how candidates sharing a merge key
        and the two blank-flag variants of a prefix combine (DecoderOptions.merge_mode,
        decoder.py:610-613, :789-791)."""
        if mode not in ("logadd", "max"):
            raise ValueError('merge_mode must be one of ("logadd", "max")')
        _lib.check(_lib.load().ctcb_set_merge_mode(self._h, 1 if mode == "max" else 0), "ctcb_set_merge_mode")

    def set_lm(self, lm, lm_weight: float = 2.0) -> None:
        """Token-level shallow fusion with a backoff n-gram model (lexicon-free
        ``beam_search_decode(..., lm=lm)``, decoder.py:178-259, :467-473,
        :753-817): ``lm`` is a :class:`paper_2310_17864_b200.lm.NGramLM` (or the
        reference's, same fields), None to detach.  Token strings are looked up
        in the model's vocabulary; blank and the silence token carry no LM
        score.  Hypothesis scores then include ``lm_weight`` × LM and the
        decode outputs carry the LM totals (``DecodeOutput.lm``)."""
        from . import lm as _lmmod
        lib = _lib.load()
        vp = ctypes.c_void_p
        if lm is None:
            _lib.check(lib.ctcb_set_lm(self._h, None, None, 0.0), "ctcb_set_lm")
            if self._lm is not None:
                lib.ctcb_lm_destroy(self._lm)
            self._lm = None
            self.lm_weight = 0.0
            return
        flat = _lmmod.flatten(lm)
        words = np.ascontiguousarray(flat.words, dtype=np.int32)
        lens = np.ascontiguousarray(flat.lengths, dtype=np.int32)
        lp = np.ascontiguousarray(flat.logprob, dtype=np.float64)
        bo = np.ascontiguousarray(flat.backoff, dtype=np.float64)
        st = np.ascontiguousarray(flat.start, dtype=np.int32)
        m = ctypes.c_void_p()
        _lib.check(lib.ctcb_lm_create(flat.order, len(lens), vp(words.ctypes.data), vp(lens.ctypes.data),
                                      vp(lp.ctypes.data), vp(bo.ctypes.data), vp(st.ctypes.data), flat.start_len,
                                      flat.eos, self.device.index, ctypes.byref(m)), "ctcb_lm_create")
        tw = np.ascontiguousarray(_lmmod.token_words(lm, self.vocab_list, self.blank_id, self.silence_index),
                                  dtype=np.int32)
        rc = lib.ctcb_set_lm(self._h, m, vp(tw.ctypes.data), float(lm_weight))
        if rc != _lib.CTCB_OK:
            lib.ctcb_lm_destroy(m)
            _lib.check(rc, "ctcb_set_lm")
        if self._lm is not None:
            lib.ctcb_lm_destroy(self._lm)
        self._lm = m
        self._lm_model = lm
        self.lm_weight = float(lm_weight)

    def set_silence(self, index: Optional[int], sil_score: float = 0.0) -> None:
        """Silence token (TokenDictionary.silence_index) and its per-emission
        bonus ``sil_score`` (decoder.py:485-486); it carries no LM score."""
        _lib.check(_lib.load().ctcb_set_silence(self._h, -1 if index is None else int(index), float(sil_score)),
                   "ctcb_set_silence")
        self.silence_index = None if index is None else int(index)
        self.sil_score = float(sil_score)
        if self._lm is not None:  # the silence column of the LM tables is the identity
            self.set_lm(self._lm_model, self.lm_weight)

    def set_beam_size_token(self, k: Optional[int]) -> None:
        """``DecoderOptions.beam_size_token``: None (default) or V searches the
        full vocabulary; K < V restricts each frame's candidates to its K best
        tokens, blank included (decoder.py:440-458)."""
        if k is not None and k < 1:
            raise ValueError("beam_size_token must be >= 1")
        _lib.check(_lib.load().ctcb_set_beam_size_token(self._h, 0 if k is None else int(k)),
                   "ctcb_set_beam_size_token")
        self.beam_size_token = None if k is None or k >= len(self.vocab_list) else int(k)

    def set_validate(self, mode) -> None:
        """Input validation fused into every decode (ctcb_set_validate), the
        checks EmissionMatrix(strict=True) runs before ctcforge decodes an
        utterance (emissions.py:128-150): True / "strict" (default), False /
        "off", or "nonstrict" (no row-normalisation check).  Failures raise the
        reference's ValueError when results are read (to_host / __call__)."""
        m = {True: 1, "strict": 1, False: 0, "off": 0, "nonstrict": 2}.get(mode)
        if m is None:
            raise ValueError("validate must be True/'strict', False/'off' or 'nonstrict'")
        _lib.check(_lib.load().ctcb_set_validate(self._h, m), "ctcb_set_validate")
        self.validate = mode

    def kernel_timing(self, enable: bool = True) -> None:
        """Record CUDA events around the beam-search kernel of every following
        decode (measurement only; see ctcb_kernel_timing)."""
        _lib.check(_lib.load().ctcb_kernel_timing(self._h, 1 if enable else 0), "ctcb_kernel_timing")

    def kernel_time(self) -> tuple[float, int, str]:
        """(summed kernel ms, timed launches, last kernel name) since kernel_timing()."""
        lib = _lib.load()
        ms, n, name = ctypes.c_double(), ctypes.c_int(), ctypes.c_char_p()
        _lib.check(lib.ctcb_kernel_time(self._h, ctypes.byref(ms), ctypes.byref(n), ctypes.byref(name)),
                   "ctcb_kernel_time")
        return ms.value, n.value, (name.value or b"").decode()

    def launch_count(self) -> int:
        """Kernels launched by this decoder's handle so far (host counter)."""
        n = ctypes.c_uint64()
        _lib.check(_lib.load().ctcb_launch_count(self._h, ctypes.byref(n)), "ctcb_launch_count")
        return int(n.value)

    def debug_counters(self) -> dict:
        """Slow-path counters of the last decode (see include/ctcb.h)."""
        lib = _lib.load()
        arr = (ctypes.c_uint64 * 8)()
        _lib.check(lib.ctcb_debug_counters(self._h, arr), "ctcb_debug_counters")
        names = ("key_ties", "exact_ties", "materializations", "materialize_steps", "radix_fallbacks",
                 "oneshot_unordered", "topk_fixups", "oneshot_fallbacks")
        return {n: int(arr[i]) for i, n in enumerate(names)}

    def debug_frames(self, log_prob: torch.Tensor, encoder_out_lens: torch.Tensor):
        """Minimum slice: (frame_map [B,T], kept [B], topk_tok [B,T,k],
        topk_val [B,T,k], blank [B,T]) device tensors after synchronisation."""
        with self._on_stream():
            return self._debug_frames(log_prob, encoder_out_lens)

    def _debug_frames(self, log_prob, encoder_out_lens):
        log_prob, lens = self._check_inputs(log_prob, encoder_out_lens)
        lib = _lib.load()
        B, T, _ = log_prob.shape
        dev = self.device
        k = self.topk
        fm = torch.full((B, max(T, 1)), -1, dtype=torch.int32, device=dev)
        kept = torch.zeros(B, dtype=torch.int32, device=dev)
        tt = torch.full((B, max(T, 1), k), -1, dtype=torch.int32, device=dev)
        tv = torch.zeros((B, max(T, 1), k), dtype=torch.float32, device=dev)
        bl = torch.zeros((B, max(T, 1)), dtype=torch.float32, device=dev)
        vp = ctypes.c_void_p
        _lib.check(lib.ctcb_debug_frames(self._h, vp(log_prob.data_ptr()), self._strides[0], self._strides[1],
                                         vp(lens.data_ptr()), B, T, self._stream(), vp(fm.data_ptr()),
                                         vp(kept.data_ptr()), vp(tt.data_ptr()), vp(tv.data_ptr()),
                                         vp(bl.data_ptr())), "ctcb_debug_frames")
        torch.cuda.synchronize(dev)
        return fm, kept, tt, tv, bl


def cuda_ctc_decoder(
    tokens: Union[str, List[str]],
    nbest: int = 1,
    beam_size: int = 10,
    blank_skip_threshold: float = _DEFAULT_BLANK_SKIP_THRESHOLD,
    **kwargs,
) -> CUCTCDecoder:
    """Build a :class:`CUCTCDecoder`.  ``tokens``: a list of token strings or
    a file with one token per line (first whitespace field); blank is index 0."""
    if isinstance(tokens, str):
        tokens = _read_vocab(tokens)
    return CUCTCDecoder(vocab_list=tokens, beam_size=beam_size, nbest=nbest,
                        blank_skip_threshold=blank_skip_threshold, **kwargs)
