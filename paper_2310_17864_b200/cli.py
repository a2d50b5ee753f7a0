"""``decode`` and ``align`` commands on the GPU: the reference's CLI callers of
the decoder and alignment paths (ctcforge cli.py:262-388, SURVEY.md §8(f1),
(f4)) with the same inputs, flags, outputs and exit codes, processing a corpus
in batched ``ctcb_decode`` / ``ctcb_align`` launches instead of one CPU call per
utterance.

    python -m paper_2310_17864_b200 align --emissions DIR|FILE --tokens FILE --refs REFS
        [--lexicon LEX] [--out OUT.jsonl] [--attribute-blanks] [--no-strict-validation]

    python -m paper_2310_17864_b200 decode --emissions DIR|FILE --tokens FILE --out OUT.jsonl
        [--config JSON] [--beam-size N] [--beam-threshold X] [--blank-skip-threshold P]
        [--nbest N] [--merge logadd|max] [--beam-size-token K] [--blank-token T] [--silence-token T]
        [--no-strict-validation] [--workers N] [--gpu-batch N] [--device D]

Inputs (emissions.py:181-253): one utterance per ``.ctce`` / ``.bin`` / ``.tsv``
file (a directory is scanned in sorted order, the utterance id is the file
stem); binary files are ``CTCE`` + version 1 + T + V (little-endian u32) + f32
rows, anything else is parsed as UTF-8 TSV.  Tokens come from a one-token-
per-line file with the blank named ``<blank>`` (else ``-``) or ``--blank-token``
(TokenDictionary.from_file, emissions.py:79-113) -- the ctcforge rule, not the
TorchAudio first-field rule of ``cuda_ctc_decoder``.

Outputs (cli.py:235-312): JSON-lines records sorted by utterance id,
``{"utt", "nbest": [{"rank", "score", "am_score", "lm_score", "token_ids",
"tokens", "words", "timesteps"}]}`` dumped with ``sort_keys=True,
ensure_ascii=False``, plus ``OUT.meta`` (total time, per-utterance times, failed
ids, decoder options).  Exit codes: 0 success, 1 when any utterance failed
(the others are still written), 2 on configuration errors.

What differs from the CPU command: the decoder is the lexicon-free CUDA search
(token-level ``--lm`` fusion and the ``--sil-score`` bonus included), so
``--lexicon`` is a configuration error (exit 2), as is ``--lm`` with a beam
above 128; TSV values are rounded to
float32, the decoder's input dtype (CTCE files are float32 already, so their
decode is bit-identical to the CPU command's); per-utterance times in the meta
file are the utterance's share of its batch (load + decode).
"""

from __future__ import annotations

import argparse
import dataclasses
import json
import logging
import os
import struct
import sys
import time
from pathlib import Path

import numpy as np

log = logging.getLogger("ctcforge")

BINARY_MAGIC = b"CTCE"          # emissions.py:18-19
BINARY_VERSION = 1
MAX_LOG_PROB = 1e-4             # emissions.py:23-24
ROW_NORM_TOL = 1e-3
EMISSION_SUFFIXES = (".ctce", ".bin", ".tsv")  # cli.py:39

_UNSET = object()

DEFAULTS = {  # cli.py:41-65
    "emissions": None, "tokens": None, "lexicon": None, "lm": None, "out": None,
    "beam_size": 10, "beam_size_token": None, "beam_threshold": 50.0, "lm_weight": 2.0,
    "word_score": 0.0, "sil_score": 0.0, "blank_skip_threshold": 1.0, "nbest": 1, "merge": "logadd",
    "workers": 1, "strict_validation": True, "blank_token": None, "silence_token": None,
    "gpu_batch": 1024, "device": 0, "refs": None, "attribute_blanks": False,
}


class ConfigError(Exception):
    pass


class EmissionFormatError(ValueError):
    """An emission file does not match the binary or TSV layout (emissions.py:32-33)."""


# --------------------------------------------------------------------------- tokens
@dataclasses.dataclass
class TokenDictionary:
    """Token inventory with a designated blank (emissions.py:36-113)."""

    tokens: tuple
    blank_index: int
    silence_index: int | None = None

    def __post_init__(self):
        self.tokens = tuple(self.tokens)
        if not self.tokens:
            raise ValueError("token dictionary is empty")
        if any(not t for t in self.tokens):
            raise ValueError("token strings must be non-empty")
        if len(set(self.tokens)) != len(self.tokens):
            raise ValueError("token strings must be unique")
        if not 0 <= self.blank_index < len(self.tokens):
            raise ValueError(f"blank_index {self.blank_index} out of range")
        if self.silence_index is not None:
            if not 0 <= self.silence_index < len(self.tokens):
                raise ValueError(f"silence_index {self.silence_index} out of range")
            if self.silence_index == self.blank_index:
                raise ValueError("silence_index must differ from blank_index")

    def __len__(self):
        return len(self.tokens)

    @classmethod
    def from_file(cls, path, blank_token=None, silence_token=None) -> "TokenDictionary":
        lines = Path(path).read_text(encoding="utf-8").splitlines()
        tokens = []
        for lineno, raw in enumerate(lines, start=1):
            tok = raw.strip()
            if not tok:
                raise EmissionFormatError(f"{path}: line {lineno}: empty token")
            tokens.append(tok)
        candidates = [blank_token] if blank_token is not None else ["<blank>", "-"]
        blank_index = next((tokens.index(c) for c in candidates if c in tokens), None)
        if blank_index is None:
            raise EmissionFormatError(f"{path}: no blank token found (looked for {', '.join(candidates)})")
        silence_index = None
        if silence_token is not None:
            if silence_token not in tokens:
                raise EmissionFormatError(f"{path}: silence token {silence_token!r} not in token file")
            silence_index = tokens.index(silence_token)
        return cls(tuple(tokens), blank_index, silence_index)


# --------------------------------------------------------------------------- emissions
def parse_emissions(path, n_tokens: int) -> np.ndarray:
    """Read one emission file as float32 [T, V] (load_emissions, emissions.py:181-253):
    format sniffed from the magic, column count checked against the token
    dictionary, non-finite values rejected."""
    path = Path(path)
    raw = path.read_bytes()
    if raw[:4] == BINARY_MAGIC:
        lp = _parse_binary(path, raw)
    else:
        lp = _parse_tsv(path, raw)
    if lp.shape[1] != n_tokens:
        raise EmissionFormatError(f"{path}: {lp.shape[1]} columns but the token dictionary has {n_tokens} tokens")
    bad = ~np.isfinite(lp)
    if bad.any():
        t, v = np.argwhere(bad)[0]
        raise EmissionFormatError(f"{path}: non-finite value at frame {t}, column {v}")
    return lp


def _parse_binary(path: Path, raw: bytes) -> np.ndarray:
    header = struct.calcsize("<4sIII")
    if len(raw) < header:
        raise EmissionFormatError(f"{path}: truncated header")
    magic, version, t, v = struct.unpack_from("<4sIII", raw)
    if version != BINARY_VERSION:
        raise EmissionFormatError(f"{path}: unsupported version {version}")
    if v == 0:
        raise EmissionFormatError(f"{path}: zero-width matrix")
    expected = header + 4 * t * v
    if len(raw) != expected:
        raise EmissionFormatError(f"{path}: expected {expected} bytes for a {t}x{v} matrix, got {len(raw)}")
    return np.frombuffer(raw, dtype="<f4", count=t * v, offset=header).reshape(t, v)


def _parse_tsv(path: Path, raw: bytes) -> np.ndarray:
    try:
        text = raw.decode("utf-8")
    except UnicodeDecodeError as exc:
        raise EmissionFormatError(f"{path}: neither CTCE binary nor UTF-8 TSV") from exc
    rows, width = [], None
    for lineno, line in enumerate(text.splitlines(), start=1):
        if not line.strip():
            continue
        fields = line.split("\t")
        if width is None:
            width = len(fields)
        elif len(fields) != width:
            raise EmissionFormatError(f"{path}: line {lineno}: expected {width} columns, got {len(fields)}")
        try:
            rows.append([float(f) for f in fields])
        except ValueError as exc:
            raise EmissionFormatError(f"{path}: line {lineno}: {exc}") from exc
    if not rows:
        return np.zeros((0, 0), dtype=np.float32)
    return np.asarray(rows, dtype=np.float64).astype(np.float32)


def write_emissions(log_probs: np.ndarray, path) -> None:
    """Binary writer (emissions.py:255-260): CTCE magic, version, T, V, f32 rows."""
    lp = np.asarray(log_probs)
    t, v = lp.shape
    with open(path, "wb") as fh:
        fh.write(struct.pack("<4sIII", BINARY_MAGIC, BINARY_VERSION, t, v))
        fh.write(lp.astype("<f4").tobytes())


# --------------------------------------------------------------------------- lexicon / transcripts
class LexiconFormatError(ValueError):
    """A lexicon file line is malformed (lexicon.py:14-15)."""


@dataclasses.dataclass
class Lexicon:
    words: list
    entries: dict  # word -> list of spellings (tuples of token indices)


def parse_lexicon(path, tokens: TokenDictionary) -> Lexicon:
    """"word token token ..." lines, '#' comments, variants per word
    (lexicon.py:87-122)."""
    path = Path(path)
    index = {tok: i for i, tok in enumerate(tokens.tokens)}
    words, entries = [], {}
    for lineno, raw in enumerate(path.read_text(encoding="utf-8").splitlines(), 1):
        line = raw.strip()
        if not line or line.startswith("#"):
            continue
        fields = line.split()
        word, spelling_toks = fields[0], fields[1:]
        if not spelling_toks:
            raise LexiconFormatError(f"{path}: line {lineno}: empty spelling")
        spelling = []
        for tok in spelling_toks:
            if tok not in index:
                raise LexiconFormatError(f"{path}: line {lineno}: unknown spelling token {tok!r}")
            spelling.append(index[tok])
        spelling = tuple(spelling)
        if word not in entries:
            entries[word] = []
            words.append(word)
        if spelling in entries[word]:
            raise LexiconFormatError(f"{path}: line {lineno}: duplicate spelling for {word!r}")
        entries[word].append(spelling)
    return Lexicon(words=words, entries=entries)


def read_refs(path) -> dict:
    """One utterance per line: "utt_id<TAB>word word word" (cli.py:182-195)."""
    refs = {}
    for lineno, line in enumerate(Path(path).read_text(encoding="utf-8").splitlines(), 1):
        if not line.strip():
            continue
        utt_id, sep, rest = line.partition("\t")
        if not utt_id or not sep:
            raise ConfigError(f"--refs: line {lineno}: expected 'utt_id<TAB>words'")
        refs[utt_id.strip()] = rest.split()
    return refs


def check_emission_matrix(lp: np.ndarray, strict: bool) -> None:
    """EmissionMatrix.__post_init__ checks (emissions.py:128-150) on the host."""
    lp = lp.astype(np.float64)
    if lp.size and lp.max() > MAX_LOG_PROB:
        t, v = np.argwhere(lp > MAX_LOG_PROB)[0]
        raise ValueError(f"log-probability above 0 at frame {t}, token {v}: {lp[t, v]:.6g}")
    if strict and lp.size:
        m = lp.max(axis=1)
        norms = m + np.log(np.exp(lp - m[:, None]).sum(axis=1))
        off = np.abs(norms) > ROW_NORM_TOL
        if off.any():
            t = int(np.argmax(off))
            raise ValueError(f"frame {t} is not normalized: log-sum-exp = {norms[t]:.6g} "
                             f"(tolerance {ROW_NORM_TOL}); pass strict=False to skip this check")


# --------------------------------------------------------------------------- config
def _merge_config(args: argparse.Namespace) -> dict:
    """CLI > --config JSON > defaults (cli.py:130-148)."""
    merged = dict(DEFAULTS)
    config_path = getattr(args, "config", _UNSET)
    if config_path not in (None, _UNSET):
        try:
            file_values = json.loads(Path(config_path).read_text(encoding="utf-8"))
        except (OSError, json.JSONDecodeError) as exc:
            raise ConfigError(f"--config: {exc}") from exc
        if not isinstance(file_values, dict):
            raise ConfigError("--config: expected a JSON object")
        for key, value in file_values.items():
            if key not in DEFAULTS and key not in ("hyps", "figure", "json"):
                raise ConfigError(f"--config: unknown key {key!r}")
            merged[key] = value
    for key in DEFAULTS:
        value = getattr(args, key, _UNSET)
        if value is not _UNSET:
            merged[key] = value
    return merged


def _device_index(dev) -> int:
    """--device: an ordinal, "cuda" (device 0) or "cuda:N"."""
    text = str(dev).strip().lower()
    if text == "cuda":
        return 0
    if text.startswith("cuda:"):
        text = text[5:]
    try:
        return int(text)
    except ValueError:
        raise ConfigError(f"--device: expected N, cuda or cuda:N, got {dev!r}") from None


def _options(cfg: dict):
    from .ctcforge_api import DecoderOptions

    try:
        return DecoderOptions(beam_size=cfg["beam_size"], beam_size_token=cfg["beam_size_token"],
                              beam_threshold=cfg["beam_threshold"], lm_weight=cfg["lm_weight"],
                              word_score=cfg["word_score"], sil_score=cfg["sil_score"],
                              blank_skip_threshold=cfg["blank_skip_threshold"], n_best=cfg["nbest"],
                              merge_mode=cfg["merge"])
    except ValueError as exc:
        raise ConfigError(str(exc)) from exc


def _discover_utterances(emissions: str) -> list:
    path = Path(emissions)
    if path.is_dir():
        files = sorted(p for p in path.iterdir() if p.suffix.lower() in EMISSION_SUFFIXES)
        if not files:
            raise ConfigError(f"--emissions: no {'/'.join(EMISSION_SUFFIXES)} files in {path}")
        return [(p.stem, p) for p in files]
    return [(path.stem, path)]


# --------------------------------------------------------------------------- decode
def cmd_decode(cfg: dict) -> int:
    for name in ("emissions", "tokens", "out"):
        if cfg[name] is None:
            raise ConfigError(f"--{name.replace('_', '-')} is required")
    for name in ("emissions", "tokens", "lexicon", "lm"):
        if cfg[name] is not None and not Path(cfg[name]).exists():
            raise ConfigError(f"--{name.replace('_', '-')}: file not found: {cfg[name]}")
    opts = _options(cfg)
    if cfg["lexicon"] is not None:
        raise ConfigError("the CUDA decoder is lexicon-free: --lexicon is not supported")
    try:
        tokens = TokenDictionary.from_file(cfg["tokens"], blank_token=cfg["blank_token"],
                                           silence_token=cfg["silence_token"])
    except ValueError as exc:
        raise ConfigError(f"--tokens: {exc}") from exc
    lm = None
    if cfg["lm"] is not None:  # cli.py:214-216: a malformed model is a configuration error
        from .lm import parse_arpa

        try:
            lm = parse_arpa(cfg["lm"])
        except ValueError as exc:
            raise ConfigError(str(exc)) from exc
    batch = int(cfg["gpu_batch"])
    if batch < 1:
        raise ConfigError("--gpu-batch must be >= 1")
    utts = _discover_utterances(cfg["emissions"])

    import torch

    from . import _lib
    from .decoder import CUCTCDecoder

    dec = CUCTCDecoder(list(tokens.tokens), blank_id=tokens.blank_index, beam_size=opts.beam_size,
                       nbest=opts.n_best, blank_skip_threshold=opts.blank_skip_threshold,
                       beam_threshold=opts.beam_threshold, device=_device_index(cfg["device"]))
    dec.set_merge_mode(opts.merge_mode)
    try:
        if tokens.silence_index is not None:
            dec.set_silence(tokens.silence_index, opts.sil_score)
        if lm is not None:
            dec.set_lm(lm, opts.lm_weight)
    except ValueError as exc:
        raise ConfigError(str(exc)) from exc
    too_wide = opts.beam_size_token is not None and opts.beam_size_token > len(tokens)
    if opts.beam_size_token is not None and not too_wide:
        dec.set_beam_size_token(opts.beam_size_token)
    strict = bool(cfg["strict_validation"])
    records, failed, times = [], [], {}
    for i0 in range(0, len(utts), batch):
        group = utts[i0:i0 + batch]
        t0 = time.perf_counter()
        lps, ids, errors = [], [], {}
        for utt_id, path in group:
            try:
                lps.append(parse_emissions(path, len(tokens)))
                ids.append(utt_id)
            except ValueError as exc:
                errors[utt_id] = str(exc)
        if lps and too_wide:  # decoder.py:124-128, per utterance
            for utt_id in ids:
                errors[utt_id] = f"beam_size_token {opts.beam_size_token} exceeds vocabulary size {len(tokens)}"
        elif lps:
            recs, errs = _decode_group(dec, tokens, ids, lps, strict, torch, _lib, opts)
            records.extend(recs)
            errors.update(errs)
        share = (time.perf_counter() - t0) / max(len(group), 1)
        for utt_id, _ in group:
            times[utt_id] = share
            if utt_id in errors:
                log.error("utterance %s failed: %s", utt_id, errors[utt_id])
                failed.append(utt_id)
    records.sort(key=lambda r: r["utt"])
    with open(cfg["out"], "w", encoding="utf-8") as fh:
        for record in records:
            fh.write(json.dumps(record, sort_keys=True, ensure_ascii=False) + "\n")
    meta = {"command": "decode", "total_time_s": sum(times.values()),
            "utterances": {u: times[u] for u in sorted(times)}, "failed": sorted(failed),
            "options": dataclasses.asdict(opts)}
    Path(cfg["out"] + ".meta").write_text(json.dumps(meta, sort_keys=True, indent=2) + "\n", encoding="utf-8")
    log.info("decoded %d utterances (%d failed)", len(records), len(failed))
    return 1 if failed else 0


def _decode_group(dec, tokens, ids, lps, strict, torch, _lib, opts):
    """Validate (EmissionMatrix checks, emissions.py:128-150) and decode one
    batch on the GPU; returns (records, {utt_id: error})."""
    import ctypes

    B, V = len(lps), len(tokens)
    T = max(max(lp.shape[0] for lp in lps), 1)
    host = torch.zeros((B, T, V), dtype=torch.float32, pin_memory=True)
    hnp = host.numpy()
    lens = np.zeros(B, dtype=np.int32)
    for b, lp in enumerate(lps):
        hnp[b, : lp.shape[0]] = lp
        lens[b] = lp.shape[0]
    dev = dec.device
    x = host.to(dev, non_blocking=True)
    lens_dev = torch.from_numpy(lens).to(dev)
    errors = {}
    # validation kernel: first offending (b, t, v); the utterance is failed,
    # masked out (length 0) and the batch re-checked
    lib = _lib.load()
    err = torch.empty(4, dtype=torch.int64, device=dev)
    while True:
        _lib.check(lib.ctcb_validate(dec._h, ctypes.c_void_p(x.data_ptr()), T * V, V,
                                     ctypes.c_void_p(lens_dev.data_ptr()), B, T, 1 if strict else 0, dec._stream(),
                                     ctypes.c_void_p(err.data_ptr())), "ctcb_validate")
        code, b, t, v = err.cpu().tolist()
        if code == 0:
            break
        lp = lps[b].astype(np.float64)
        if code == 1:
            errors[ids[b]] = f"non-finite log-probability at frame {t}, token {v}"
        elif code == 2:
            errors[ids[b]] = f"log-probability above 0 at frame {t}, token {v}: {lp[t, v]:.6g}"
        else:
            m = lp[t].max()
            norm = m + np.log(np.exp(lp[t] - m).sum())
            errors[ids[b]] = (f"frame {t} is not normalized: log-sum-exp = {norm:.6g} (tolerance {ROW_NORM_TOL}); "
                              "pass strict=False to skip this check")
        lens[b] = 0
        lens_dev[b] = 0
    for b in range(B):
        if lens[b] == 0 and ids[b] not in errors:
            errors[ids[b]] = "empty emissions"  # decoder.py:117-118
    out = dec.decode(x, lens_dev, timesteps=True)
    status = out.status.cpu().numpy()
    counts = out.counts.cpu().numpy()
    lengths = out.lengths.cpu().numpy()
    scores = out.scores.cpu().numpy()
    lmax = int(lengths.max()) if lengths.size else 0
    toks = out.tokens[:, :, :lmax].cpu().numpy()
    ts = out.timesteps[:, :, :lmax].cpu().numpy()
    lms = out.lm.cpu().numpy() if out.lm is not None else None
    sil = tokens.silence_index
    records = []
    names = tokens.tokens
    for b in range(B):
        if ids[b] in errors:
            continue
        if status[b] == _lib.UTT_BEAM_DIED:
            K = dec.beam_size_token or V
            errors[ids[b]] = (f"beam died at frame {int(lengths[b, 0])}: no extension survives "
                              f"(beam_size_token={K} may be too small)")
            continue
        nbest = []
        for r in range(int(counts[b])):
            n = int(lengths[b, r])
            ti = toks[b, r, :n].tolist()
            sc = float(scores[b, r])
            lm_v = float(lms[b, r]) if lms is not None else 0.0
            # am_score = score - lm_weight * lm - bonuses (decoder.py:805-812)
            bonuses = opts.word_score * 0 + opts.sil_score * (ti.count(sil) if sil is not None else 0)
            am = sc - (opts.lm_weight * lm_v if lms is not None else 0.0) - bonuses
            nbest.append({"rank": r, "score": sc, "am_score": am, "lm_score": lm_v, "token_ids": ti,
                          "tokens": [names[i] for i in ti], "words": [], "timesteps": ts[b, r, :n].tolist()})
        records.append({"utt": ids[b], "nbest": nbest})
    return records, errors


# --------------------------------------------------------------------------- align
def cmd_align(cfg: dict) -> int:
    """Force-align transcripts to emissions (cli.py:327-388) with one
    ``ctcb_align`` launch per batch of utterances; records in utterance order,
    an ``{"utt", "error"}`` record per failed utterance."""
    for name in ("emissions", "tokens", "refs"):
        if cfg[name] is None:
            raise ConfigError(f"--{name.replace('_', '-')} is required")
    for name in ("emissions", "tokens", "refs", "lexicon"):
        if cfg[name] is not None and not Path(cfg[name]).exists():
            raise ConfigError(f"--{name.replace('_', '-')}: file not found: {cfg[name]}")
    try:
        tokens = TokenDictionary.from_file(cfg["tokens"], blank_token=cfg["blank_token"],
                                           silence_token=cfg["silence_token"])
    except ValueError as exc:
        raise ConfigError(f"--tokens: {exc}") from exc
    lexicon = parse_lexicon(cfg["lexicon"], tokens) if cfg["lexicon"] else None
    refs = read_refs(cfg["refs"])
    utts = _discover_utterances(cfg["emissions"])
    from . import align as galign

    strict = bool(cfg["strict_validation"])
    batch = int(cfg["gpu_batch"])
    failed = 0
    out = sys.stdout if cfg["out"] is None else open(cfg["out"], "w", encoding="utf-8")
    index = {t: i for i, t in enumerate(tokens.tokens)}
    try:
        for i0 in range(0, len(utts), batch):
            group = utts[i0:i0 + batch]
            prepared, results = [], {}
            for utt_id, path in group:
                try:
                    if utt_id not in refs:
                        raise ValueError(f"no transcript for {utt_id} in --refs")
                    transcript = refs[utt_id]
                    lp = parse_emissions(path, len(tokens))
                    check_emission_matrix(lp, strict)
                    if lexicon is not None:
                        targets = []
                        for word in transcript:
                            variants = lexicon.entries.get(word)
                            if not variants:
                                raise ValueError(f"word {word!r} is not in the lexicon")
                            targets.extend(variants[0])
                    else:
                        targets = []
                        for tok in transcript:  # TokenDictionary.index (emissions.py:69-73)
                            if tok not in index:
                                raise KeyError(f"unknown token: {tok!r}")
                            targets.append(index[tok])
                    prepared.append((utt_id, transcript, lp, targets))
                except Exception as exc:  # noqa: BLE001 - per-utterance failure, as cli.py:339-344
                    results[utt_id] = str(exc)
            if prepared:
                aligned = galign.forced_align_batch([p[2] for p in prepared], [p[3] for p in prepared], tokens,
                                                    device=_device_index(cfg["device"]), raise_errors=False)
                for (utt_id, transcript, _, _), r in zip(prepared, aligned):
                    results[utt_id] = (transcript, r) if not isinstance(r, str) else r
            for utt_id, _ in group:
                r = results[utt_id]
                try:
                    if isinstance(r, str):
                        raise ValueError(r)
                    records = _align_records(cfg, tokens, lexicon, utt_id, *r, galign)
                except Exception as exc:  # noqa: BLE001
                    out.write(json.dumps({"utt": utt_id, "error": str(exc)}, sort_keys=True, ensure_ascii=False) + "\n")
                    log.error("utterance %s failed: %s", utt_id, exc)
                    failed += 1
                    continue
                for record in records:
                    out.write(json.dumps(record, sort_keys=True, ensure_ascii=False) + "\n")
    finally:
        if out is not sys.stdout:
            out.close()
    return 1 if failed else 0


def _align_records(cfg, tokens, lexicon, utt_id, transcript, result, galign) -> list:
    import math

    spans = galign.attribute_blanks(result) if cfg["attribute_blanks"] else result.spans
    records = [{"utt": utt_id, "token": tokens.tokens[sp.token], "start": sp.start_frame, "end": sp.end_frame,
                "score": sp.score, "prob": math.exp(sp.score)} for sp in spans]
    if lexicon is not None:
        for ws in galign.align_words(result, tokens, transcript, lexicon):
            records.append({"utt": utt_id, "word": ws.word, "start": ws.start_frame, "end": ws.end_frame,
                            "score": ws.score, "prob": math.exp(ws.score)})
    return records


# --------------------------------------------------------------------------- argparse
def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="paper_2310_17864_b200",
                                     description="CTC beam-search decoding on the GPU (ctcforge decode)")
    sub = parser.add_subparsers(dest="command", required=True)
    p = sub.add_parser("decode", help="beam-search decode emission files")
    p.add_argument("--config", default=_UNSET, help="JSON config file")
    p.add_argument("--tokens", default=_UNSET, help="token file, one token per line")
    p.add_argument("--blank-token", default=_UNSET, dest="blank_token")
    p.add_argument("--silence-token", default=_UNSET, dest="silence_token")
    p.add_argument("--strict-validation", action=argparse.BooleanOptionalAction, default=_UNSET,
                   dest="strict_validation")
    p.add_argument("--lexicon", default=_UNSET)
    p.add_argument("--lm", default=_UNSET)
    p.add_argument("--beam-size", type=int, default=_UNSET, dest="beam_size")
    p.add_argument("--beam-size-token", type=int, default=_UNSET, dest="beam_size_token")
    p.add_argument("--beam-threshold", type=float, default=_UNSET, dest="beam_threshold")
    p.add_argument("--lm-weight", type=float, default=_UNSET, dest="lm_weight")
    p.add_argument("--word-score", type=float, default=_UNSET, dest="word_score")
    p.add_argument("--sil-score", type=float, default=_UNSET, dest="sil_score")
    p.add_argument("--blank-skip-threshold", type=float, default=_UNSET, dest="blank_skip_threshold",
                   help="drop frames with at least this blank probability (1.0 disables)")
    p.add_argument("--nbest", type=int, default=_UNSET)
    p.add_argument("--merge", choices=["max", "logadd"], default=_UNSET)
    p.add_argument("--emissions", default=_UNSET, help="emission file or directory")
    p.add_argument("--out", default=_UNSET, help="output JSON-lines path (required)")
    p.add_argument("--workers", type=int, default=_UNSET, help="accepted for compatibility (the GPU batches)")
    p.add_argument("--gpu-batch", type=int, default=_UNSET, dest="gpu_batch", help="utterances per launch")
    p.add_argument("--device", default=_UNSET, help="CUDA device: N, cuda or cuda:N")

    p = sub.add_parser("align", help="force-align transcripts to emissions")
    p.add_argument("--config", default=_UNSET, help="JSON config file")
    p.add_argument("--tokens", default=_UNSET, help="token file, one token per line")
    p.add_argument("--blank-token", default=_UNSET, dest="blank_token")
    p.add_argument("--silence-token", default=_UNSET, dest="silence_token")
    p.add_argument("--strict-validation", action=argparse.BooleanOptionalAction, default=_UNSET,
                   dest="strict_validation")
    p.add_argument("--emissions", default=_UNSET, help="emission file or directory")
    p.add_argument("--refs", default=_UNSET, help="transcripts: utt_id<TAB>words")
    p.add_argument("--lexicon", default=_UNSET, help="word mode: spell transcript words through this lexicon")
    p.add_argument("--out", default=_UNSET, help="output JSON-lines path (default: stdout)")
    p.add_argument("--attribute-blanks", action=argparse.BooleanOptionalAction, default=_UNSET,
                   dest="attribute_blanks", help="widen spans so blanks attach to the preceding token")
    p.add_argument("--gpu-batch", type=int, default=_UNSET, dest="gpu_batch", help="utterances per launch")
    p.add_argument("--device", default=_UNSET, help="CUDA device: N, cuda or cuda:N")
    return parser


def main(argv=None) -> int:
    level = os.environ.get("CTCFORGE_LOG", "WARNING").upper()
    if not isinstance(getattr(logging, level, None), int):
        level = "WARNING"
    logging.basicConfig(level=level, format="%(levelname)s %(name)s: %(message)s")
    args = build_parser().parse_args(argv)
    try:
        cfg = _merge_config(args)
        if args.command == "align":
            return cmd_align(cfg)
        return cmd_decode(cfg)
    except ConfigError as exc:
        print(f"ctcforge {args.command}: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
