"""One process, several GPUs: ``MultiDeviceDecoder``.

Utterances are independent, so a batch splits into per-device work with no
data-path collective.  The batch is cut into consecutive utterance ranges with
balanced Σ len (:func:`shard.balanced_ranges`): a range of a [B, T, V] tensor
is a view, so no host-side gather is needed, and each device's kernel orders
its own range longest-first.  One host thread per device drives that device's
decoder (its own handle, stream and workspace) through the same entry points as
the single-device façade; results are reassembled in batch order on the host.

    dec = MultiDeviceDecoder(tokens, devices=[0, 1, 2, 3], beam_size=10)
    hyps = dec(log_probs, encoder_out_lens)   # CPU (pinned) or CUDA tensors

Host (CPU) inputs go through ``ctcb_decode_host_async`` per device (each
device reads its range straight from the pinned buffer).  CUDA inputs on
device s are decoded in place on s for s's own range, and the other ranges are
copied peer-to-peer to their device first.  Errors carry the utterance's
index in the whole batch; when several ranges fail, the first failing
utterance in batch order is reported, as the single-device decoder does.
"""

from __future__ import annotations

import threading
from typing import List, Optional, Sequence

import torch

from .decoder import CUCTCDecoder, CUCTCHypothesis, cuda_ctc_decoder
from .shard import balanced_ranges

__all__ = ["MultiDeviceDecoder"]


class MultiDeviceDecoder:
    """A :class:`CUCTCDecoder` per device over consecutive length-balanced
    utterance ranges.  ``devices`` may repeat an index (two decoders, two
    streams on one GPU)."""

    def __init__(self, tokens, devices: Optional[Sequence[int]] = None, nbest: int = 1, beam_size: int = 10,
                 blank_skip_threshold: float = 0.95, **kwargs):
        if kwargs.get("cuda_stream") is not None:
            raise ValueError("MultiDeviceDecoder creates one stream per device; cuda_stream is not accepted")
        kwargs.pop("cuda_stream", None)
        kwargs.pop("device", None)
        if devices is None:
            devices = list(range(torch.cuda.device_count()))
        devices = [int(d) for d in devices]
        if not devices:
            raise ValueError("at least one device is required")
        self.devices = devices
        self.decoders: List[CUCTCDecoder] = []
        for d in devices:
            stream = torch.cuda.Stream(device=d)
            self.decoders.append(cuda_ctc_decoder(tokens, nbest=nbest, beam_size=beam_size,
                                                  blank_skip_threshold=blank_skip_threshold, device=d,
                                                  cuda_stream=stream, **kwargs))
        self.last_ranges: list[tuple[int, int]] = []

    # options apply to every device's decoder
    def set_merge_mode(self, mode: str) -> None:
        for dec in self.decoders:
            dec.set_merge_mode(mode)

    def set_beam_size_token(self, k: Optional[int]) -> None:
        for dec in self.decoders:
            dec.set_beam_size_token(k)

    def set_silence(self, index: Optional[int], sil_score: float = 0.0) -> None:
        for dec in self.decoders:
            dec.set_silence(index, sil_score)

    def set_lm(self, lm, lm_weight: float = 2.0) -> None:
        """Attach a token-level n-gram model to every device's decoder (each
        device builds its own context x token tables)."""
        for dec in self.decoders:
            dec.set_lm(lm, lm_weight)

    def _run_host(self, dec: CUCTCDecoder, lp: torch.Tensor, lens, b0: int):
        B = lp.shape[0]
        chunks = max(1, min(16, B // 256))
        out = []
        for _, _, tokens, lengths, scores, counts in dec._decode_host_chunks(lp, lens, chunks, offset=b0):
            out.extend(dec._hypotheses(tokens, lengths, scores, counts))
        return out

    def _run_device(self, dec: CUCTCDecoder, lp: torch.Tensor, lens: torch.Tensor, b0: int,
                    ready: "torch.cuda.Event"):
        """`ready` was recorded on the CALLER's current stream of the input's
        device (streams are thread-local: this may run on a worker thread,
        whose current stream is the default one), so the decode -- or the
        peer copy -- is ordered after the producer of `lp`, whatever stream
        produced it."""
        with torch.cuda.device(dec.device):
            dec.cuda_stream.wait_event(ready)
            if lp.device != dec.device:
                # peer copy on the target device's stream
                with torch.cuda.stream(dec.cuda_stream):
                    lp = lp.to(dec.device, non_blocking=True)
                    lens = lens.to(dec.device, non_blocking=True)
            out = dec.decode(lp, lens, offset=b0)
            tokens, _, lengths, scores, counts = dec.to_host(out, offset=b0)
            return dec._hypotheses(tokens, lengths, scores, counts)

    def __call__(self, log_prob: torch.Tensor, encoder_out_lens) -> List[List[CUCTCHypothesis]]:
        if not isinstance(log_prob, torch.Tensor) or log_prob.dim() != 3:
            raise ValueError("log_prob must be a 3-D tensor [batch, frames, tokens]")
        B = log_prob.shape[0]
        lens_t = encoder_out_lens if isinstance(encoder_out_lens, torch.Tensor) else torch.as_tensor(encoder_out_lens)
        if lens_t.dim() != 1 or lens_t.shape[0] != B:
            raise ValueError("encoder_out_lens must be a 1-D tensor with one length per utterance")
        lens_cpu = lens_t.cpu()
        ranges = balanced_ranges(lens_cpu.numpy(), len(self.decoders))
        self.last_ranges = ranges
        on_host = not log_prob.is_cuda
        ready = None
        if not on_host:  # recorded here, on the calling thread's current stream
            ready = torch.cuda.Event()
            ready.record(torch.cuda.current_stream(log_prob.device))
            if lens_t.is_cuda and lens_t.device != log_prob.device:
                raise ValueError("log_prob and encoder_out_lens must be on the same device")
        results: list = [None] * len(ranges)
        errors: list = [None] * len(ranges)

        def work(i: int) -> None:
            b0, b1 = ranges[i]
            if b1 <= b0:
                results[i] = []
                return
            dec = self.decoders[i]
            try:
                if on_host:
                    results[i] = self._run_host(dec, log_prob[b0:b1], lens_cpu[b0:b1], b0)
                else:
                    results[i] = self._run_device(dec, log_prob[b0:b1], lens_t[b0:b1], b0, ready)
            except BaseException as exc:  # re-raised on the calling thread
                errors[i] = exc

        threads = [threading.Thread(target=work, args=(i,), daemon=True) for i in range(1, len(ranges))]
        for t in threads:
            t.start()
        work(0)
        for t in threads:
            t.join()
        for exc in errors:  # ranges are in batch order: the first failure is the first failing utterance
            if exc is not None:
                raise exc
        out: List[List[CUCTCHypothesis]] = []
        for r in results:
            out.extend(r)
        return out
