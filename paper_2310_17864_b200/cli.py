"""``decode`` and ``align`` commands on the GPU: drop-ins for the reference's
CLI callers of the decoder and alignment paths (ctcforge cli.py:262-388,
SURVEY.md §8(f1), (f4)) -- same inputs, flags, output records and exit codes --
that process a corpus in batched ``ctcb_decode`` / ``ctcb_align`` launches
instead of one CPU call per utterance.

    python -m paper_2310_17864_b200 align --emissions DIR|FILE --tokens FILE --refs REFS
        [--lexicon LEX] [--out OUT.jsonl] [--attribute-blanks] [--no-strict-validation]

    python -m paper_2310_17864_b200 decode --emissions DIR|FILE --tokens FILE --out OUT.jsonl
        [--config JSON] [--beam-size N] [--beam-threshold X] [--blank-skip-threshold P]
        [--nbest N] [--merge logadd|max] [--beam-size-token K] [--blank-token T] [--silence-token T]
        [--lm ARPA] [--lm-weight W] [--sil-score S] [--no-strict-validation] [--gpu-batch N] [--device D]

Inputs (emissions.py:181-253): one utterance per ``.ctce`` / ``.bin`` / ``.tsv``
file (a directory is taken in sorted order; the utterance id is the file
stem).  CTCE files (``CTCE`` magic, version 1, T, V as little-endian u32, then
f32 rows) are memory-mapped and their rows copied straight into the pinned
[B, T, V] batch that goes to the GPU; anything else is read as UTF-8 TSV.
Tokens: one per line, the whole stripped line, blank ``<blank>`` (else ``-``)
or ``--blank-token`` -- ctcforge's rule (emissions.py:79-113), not the
TorchAudio first-field rule of ``cuda_ctc_decoder``.

Outputs (cli.py:235-312): JSON-lines records sorted by utterance id,
``{"utt", "nbest": [{"rank", "score", "am_score", "lm_score", "token_ids",
"tokens", "words", "timesteps"}]}`` (``sort_keys=True, ensure_ascii=False``),
plus ``OUT.meta`` (total time, per-utterance times, failed ids, decoder
options).  Exit codes: 0 success, 1 when an utterance failed (the others are
still written), 2 on configuration errors.

What differs from the CPU command: the search is the lexicon-free CUDA
decoder (token-level ``--lm`` fusion and the ``--sil-score`` bonus included),
so ``--lexicon`` is a configuration error for ``decode`` (exit 2), as is
``--lm`` with a beam above 128; TSV values are rounded to float32, the
decoder's input dtype (CTCE files are float32 already, so their decode is
bit-identical to the CPU command's); an utterance's time in the meta file is
its share of its batch (load + decode).
"""

from __future__ import annotations

import argparse
import dataclasses
import json
import logging
import math
import mmap
import os
import struct
import sys
import time
from collections import ChainMap
from pathlib import Path

import numpy as np

# records of failed utterances go to the reference's logger name
log = logging.getLogger("ctcforge")

CTCE_HEADER = struct.Struct("<4sIII")   # magic, version, frames, columns (emissions.py:18-19)
CTCE_MAGIC = b"CTCE"
CTCE_VERSION = 1
MAX_LOG_PROB = 1e-4                     # EmissionMatrix limits (emissions.py:23-24)
ROW_NORM_TOL = 1e-3
EMISSION_SUFFIXES = (".ctce", ".bin", ".tsv")

_UNSET = object()

# every setting a command reads, with its default (cli.py:41-65's keys; the
# last four are GPU-specific)
SETTINGS = {
    "emissions": None, "tokens": None, "lexicon": None, "lm": None, "out": None, "refs": None,
    "beam_size": 10, "beam_size_token": None, "beam_threshold": 50.0, "lm_weight": 2.0,
    "word_score": 0.0, "sil_score": 0.0, "blank_skip_threshold": 1.0, "nbest": 1, "merge": "logadd",
    "strict_validation": True, "blank_token": None, "silence_token": None, "attribute_blanks": False,
    "workers": 1, "gpu_batch": 1024, "device": 0,
}
# keys of the reference's `evaluate` command that may sit in a shared config file
_FOREIGN_KEYS = frozenset({"hyps", "figure", "json"})


class ConfigError(Exception):
    """Bad flags, files or options: exit code 2."""


class EmissionFormatError(ValueError):
    """An emission file matches neither the CTCE nor the TSV layout."""


class LexiconFormatError(ValueError):
    """A malformed lexicon line."""


# =========================================================================== settings
def resolve_settings(args: argparse.Namespace) -> dict:
    """Layered settings: command-line flags over the ``--config`` JSON object
    over the defaults (cli.py:130-148).  Unknown keys in the file are errors."""
    layers = [{k: v for k, v in vars(args).items() if k in SETTINGS and v is not _UNSET}]
    path = getattr(args, "config", _UNSET)
    if path not in (None, _UNSET):
        try:
            loaded = json.loads(Path(path).read_text(encoding="utf-8"))
        except (OSError, json.JSONDecodeError) as exc:
            raise ConfigError(f"--config: {exc}") from exc
        if not isinstance(loaded, dict):
            raise ConfigError("--config: expected a JSON object")
        stray = next((k for k in loaded if k not in SETTINGS and k not in _FOREIGN_KEYS), None)
        if stray is not None:
            raise ConfigError(f"--config: unknown key {stray!r}")
        layers.append(loaded)
    return dict(ChainMap(*layers, SETTINGS))


def _require(cfg: dict, *names: str) -> None:
    missing = next((n for n in names if cfg[n] is None), None)
    if missing is not None:
        raise ConfigError(f"--{missing.replace('_', '-')} is required")


def _must_exist(cfg: dict, *names: str) -> None:
    for n in names:
        if cfg[n] is not None and not os.path.exists(cfg[n]):
            raise ConfigError(f"--{n.replace('_', '-')}: file not found: {cfg[n]}")


def _device_index(dev) -> int:
    """--device: an ordinal, ``cuda`` (device 0) or ``cuda:N``."""
    spec = str(dev).strip().lower()
    spec = "0" if spec == "cuda" else spec.removeprefix("cuda:")
    if not spec.isdigit():
        raise ConfigError(f"--device: expected N, cuda or cuda:N, got {dev!r}")
    return int(spec)


def _decoder_options(cfg: dict):
    from .ctcforge_api import DecoderOptions

    fields = dict(beam_size="beam_size", beam_size_token="beam_size_token", beam_threshold="beam_threshold",
                  lm_weight="lm_weight", word_score="word_score", sil_score="sil_score",
                  blank_skip_threshold="blank_skip_threshold", n_best="nbest", merge_mode="merge")
    try:
        return DecoderOptions(**{opt: cfg[key] for opt, key in fields.items()})
    except ValueError as exc:
        raise ConfigError(str(exc)) from exc


def _utterances(spec: str) -> list:
    """(utterance id, path) pairs: a single file, or a directory's emission
    files in sorted order."""
    root = Path(spec)
    if not root.is_dir():
        return [(root.stem, root)]
    found = sorted(p for p in root.iterdir() if p.suffix.lower() in EMISSION_SUFFIXES)
    if not found:
        raise ConfigError(f"--emissions: no {'/'.join(EMISSION_SUFFIXES)} files in {root}")
    return [(p.stem, p) for p in found]


# =========================================================================== tokens
@dataclasses.dataclass
class TokenDictionary:
    """Acoustic tokens with a designated blank and an optional silence
    (the contract of emissions.py:36-113, same messages)."""

    tokens: tuple
    blank_index: int
    silence_index: int | None = None

    def __post_init__(self):
        self.tokens = tuple(self.tokens)
        n = len(self.tokens)
        problems = (
            (n == 0, "token dictionary is empty"),
            (not all(self.tokens), "token strings must be non-empty"),
            (len(set(self.tokens)) != n, "token strings must be unique"),
            (not 0 <= self.blank_index < n, f"blank_index {self.blank_index} out of range"),
            (self.silence_index is not None and not 0 <= self.silence_index < n,
             f"silence_index {self.silence_index} out of range"),
            (self.silence_index is not None and self.silence_index == self.blank_index,
             "silence_index must differ from blank_index"),
        )
        for bad, msg in problems:
            if bad:
                raise ValueError(msg)

    def __len__(self) -> int:
        return len(self.tokens)

    @classmethod
    def from_file(cls, path, blank_token=None, silence_token=None) -> "TokenDictionary":
        names = [line.strip() for line in Path(path).read_text(encoding="utf-8").splitlines()]
        if "" in names:
            raise EmissionFormatError(f"{path}: line {names.index('') + 1}: empty token")
        where = {t: i for i, t in reversed(list(enumerate(names)))}  # first occurrence
        wanted = ["<blank>", "-"] if blank_token is None else [blank_token]
        blank = next((where[c] for c in wanted if c in where), None)
        if blank is None:
            raise EmissionFormatError(f"{path}: no blank token found (looked for {', '.join(wanted)})")
        if silence_token is not None and silence_token not in where:
            raise EmissionFormatError(f"{path}: silence token {silence_token!r} not in token file")
        return cls(tuple(names), blank, None if silence_token is None else where[silence_token])


# =========================================================================== emissions
class EmissionFile:
    """One utterance's emissions: the header of a CTCE file (rows stay in
    the memory-mapped file until :meth:`copy_to`), or a parsed TSV matrix."""

    def __init__(self, path: Path):
        self.path = Path(path)
        self._map = None
        self._rows = None
        with open(self.path, "rb") as fh:
            head = fh.read(4)
            if head == CTCE_MAGIC:
                fh.seek(0, os.SEEK_END)
                size = fh.tell()
                self._open_ctce(fh, size)
            else:
                fh.seek(0)
                self._rows = self._read_tsv(fh.read())
        self.frames, self.columns = (self._rows.shape if self._rows is not None else self._shape)

    def _open_ctce(self, fh, size: int) -> None:
        if size < CTCE_HEADER.size:
            raise EmissionFormatError(f"{self.path}: truncated header")
        fh.seek(0)
        _, version, t, v = CTCE_HEADER.unpack(fh.read(CTCE_HEADER.size))
        if version != CTCE_VERSION:
            raise EmissionFormatError(f"{self.path}: unsupported version {version}")
        if v == 0:
            raise EmissionFormatError(f"{self.path}: zero-width matrix")
        need = CTCE_HEADER.size + 4 * t * v
        if size != need:
            raise EmissionFormatError(f"{self.path}: expected {need} bytes for a {t}x{v} matrix, got {size}")
        self._shape = (t, v)
        if t:
            self._map = mmap.mmap(fh.fileno(), 0, access=mmap.ACCESS_READ)

    def _read_tsv(self, raw: bytes) -> np.ndarray:
        try:
            text = raw.decode("utf-8")
        except UnicodeDecodeError as exc:
            raise EmissionFormatError(f"{self.path}: neither CTCE binary nor UTF-8 TSV") from exc
        rows = []
        for lineno, line in ((k, s) for k, s in enumerate(text.splitlines(), start=1) if s.strip()):
            cells = line.split("\t")
            if rows and len(cells) != len(rows[0]):
                raise EmissionFormatError(f"{self.path}: line {lineno}: expected {len(rows[0])} columns, "
                                          f"got {len(cells)}")
            try:
                rows.append([float(c) for c in cells])
            except ValueError as exc:
                raise EmissionFormatError(f"{self.path}: line {lineno}: {exc}") from exc
        return np.array(rows, dtype=np.float64).astype(np.float32) if rows else np.zeros((0, 0), np.float32)

    def rows(self) -> np.ndarray:
        """float32 [T, V] (a read-only view of the mapped file for CTCE)."""
        if self._rows is not None:
            return self._rows
        if self._map is None:
            return np.zeros(self._shape, dtype=np.float32)
        return np.frombuffer(self._map, dtype="<f4", count=self.frames * self.columns,
                             offset=CTCE_HEADER.size).reshape(self.frames, self.columns)

    def check(self, n_tokens: int) -> "EmissionFile":
        """Column count against the token dictionary; finite values only."""
        if self.columns != n_tokens:
            raise EmissionFormatError(f"{self.path}: {self.columns} columns but the token dictionary has "
                                      f"{n_tokens} tokens")
        x = self.rows()
        finite = np.isfinite(x)
        if not finite.all():
            t, v = np.argwhere(~finite)[0]
            raise EmissionFormatError(f"{self.path}: non-finite value at frame {t}, column {v}")
        return self

    def copy_to(self, dst: np.ndarray) -> None:
        dst[: self.frames] = self.rows()

    def close(self) -> None:
        if self._map is not None:
            self._map.close()
            self._map = None


def parse_emissions(path, n_tokens: int) -> np.ndarray:
    """float32 [T, V] of one emission file (load_emissions, emissions.py:181-253)."""
    em = EmissionFile(path).check(n_tokens)
    try:
        return np.array(em.rows())
    finally:
        em.close()


def write_emissions(log_probs: np.ndarray, path) -> None:
    """CTCE writer (emissions.py:255-260)."""
    x = np.asarray(log_probs)
    with open(path, "wb") as fh:
        fh.write(CTCE_HEADER.pack(CTCE_MAGIC, CTCE_VERSION, *x.shape))
        fh.write(np.ascontiguousarray(x, dtype="<f4").tobytes())


def check_emission_matrix(lp: np.ndarray, strict: bool) -> None:
    """EmissionMatrix.__post_init__'s range and normalisation checks
    (emissions.py:128-150), same messages."""
    x = np.asarray(lp, dtype=np.float64)
    if not x.size:
        return
    over = np.argwhere(x > MAX_LOG_PROB)
    if len(over):
        t, v = over[0]
        raise ValueError(f"log-probability above 0 at frame {t}, token {v}: {x[t, v]:.6g}")
    if strict:
        peak = x.max(axis=1)
        lse = peak + np.log(np.exp(x - peak[:, None]).sum(axis=1))
        off = np.flatnonzero(np.abs(lse) > ROW_NORM_TOL)
        if off.size:
            t = int(off[0])
            raise ValueError(f"frame {t} is not normalized: log-sum-exp = {lse[t]:.6g} "
                             f"(tolerance {ROW_NORM_TOL}); pass strict=False to skip this check")


# =========================================================================== lexicon / transcripts
@dataclasses.dataclass
class Lexicon:
    words: list
    entries: dict  # word -> spellings (tuples of token indices), file order


def parse_lexicon(path, tokens: TokenDictionary) -> Lexicon:
    """``word tok tok ...`` lines, ``#`` comments, several spellings per word
    (lexicon.py:87-122's format and messages)."""
    index = {t: i for i, t in enumerate(tokens.tokens)}
    entries: dict = {}
    for lineno, line in enumerate(Path(path).read_text(encoding="utf-8").splitlines(), start=1):
        fields = line.split()
        if not fields or fields[0].startswith("#"):
            continue
        word, spelled = fields[0], fields[1:]
        if not spelled:
            raise LexiconFormatError(f"{path}: line {lineno}: empty spelling")
        unknown = next((t for t in spelled if t not in index), None)
        if unknown is not None:
            raise LexiconFormatError(f"{path}: line {lineno}: unknown spelling token {unknown!r}")
        variants = entries.setdefault(word, [])
        spelling = tuple(index[t] for t in spelled)
        if spelling in variants:
            raise LexiconFormatError(f"{path}: line {lineno}: duplicate spelling for {word!r}")
        variants.append(spelling)
    return Lexicon(words=list(entries), entries=entries)


def read_refs(path) -> dict:
    """Transcripts, ``utt_id<TAB>word word ...`` per line (cli.py:182-195)."""
    refs = {}
    for lineno, line in enumerate(Path(path).read_text(encoding="utf-8").splitlines(), start=1):
        if not line.strip():
            continue
        utt, tab, words = line.partition("\t")
        if not (utt and tab):
            raise ConfigError(f"--refs: line {lineno}: expected 'utt_id<TAB>words'")
        refs[utt.strip()] = words.split()
    return refs


def _record_line(record: dict) -> str:
    return json.dumps(record, sort_keys=True, ensure_ascii=False) + "\n"


# =========================================================================== decode
def cmd_decode(cfg: dict) -> int:
    _require(cfg, "emissions", "tokens", "out")
    _must_exist(cfg, "emissions", "tokens", "lexicon", "lm")
    opts = _decoder_options(cfg)
    if cfg["lexicon"] is not None:
        raise ConfigError("the CUDA decoder is lexicon-free: --lexicon is not supported")
    tokens = _token_dictionary(cfg)
    lm = None
    if cfg["lm"] is not None:  # a malformed model is a configuration error (cli.py:214-216)
        from .lm import parse_arpa

        try:
            lm = parse_arpa(cfg["lm"])
        except ValueError as exc:
            raise ConfigError(str(exc)) from exc
    per_launch = int(cfg["gpu_batch"])
    if per_launch < 1:
        raise ConfigError("--gpu-batch must be >= 1")
    utts = _utterances(cfg["emissions"])
    job = _DecodeJob(cfg, opts, tokens, lm)
    for k in range(0, len(utts), per_launch):
        job.run_batch(utts[k: k + per_launch])
    return job.finish(cfg["out"])


def _token_dictionary(cfg: dict) -> TokenDictionary:
    try:
        return TokenDictionary.from_file(cfg["tokens"], blank_token=cfg["blank_token"],
                                         silence_token=cfg["silence_token"])
    except ValueError as exc:
        raise ConfigError(f"--tokens: {exc}") from exc


class _DecodeJob:
    """One CUDA decoder for the whole corpus; per batch: map / parse the
    files, copy their rows into one pinned [B, T, V] buffer, decode with the
    input checks fused in (ctcb_set_validate), and build the records."""

    def __init__(self, cfg: dict, opts, tokens: TokenDictionary, lm):
        import torch

        from .decoder import CUCTCDecoder

        self.torch = torch
        self.opts, self.tokens = opts, tokens
        self.strict = bool(cfg["strict_validation"])
        self.dec = CUCTCDecoder(list(tokens.tokens), blank_id=tokens.blank_index, beam_size=opts.beam_size,
                                nbest=opts.n_best, blank_skip_threshold=opts.blank_skip_threshold,
                                beam_threshold=opts.beam_threshold, device=_device_index(cfg["device"]))
        self.dec.set_merge_mode(opts.merge_mode)
        try:
            if tokens.silence_index is not None:
                self.dec.set_silence(tokens.silence_index, opts.sil_score)
            if lm is not None:
                self.dec.set_lm(lm, opts.lm_weight)
        except ValueError as exc:
            raise ConfigError(str(exc)) from exc
        # beam_size_token > V fails every utterance (decoder.py:124-128)
        self.token_limit_error = None
        if opts.beam_size_token is not None:
            if opts.beam_size_token > len(tokens):
                self.token_limit_error = (f"beam_size_token {opts.beam_size_token} exceeds vocabulary size "
                                          f"{len(tokens)}")
            else:
                self.dec.set_beam_size_token(opts.beam_size_token)
        self.records: list = []
        self.failed: list = []
        self.seconds: dict = {}

    def run_batch(self, group: list) -> None:
        t0 = time.perf_counter()
        errors, files = {}, []
        for utt, path in group:
            try:
                files.append((utt, EmissionFile(path).check(len(self.tokens))))
            except ValueError as exc:
                errors[utt] = str(exc)
        if files and self.token_limit_error:
            errors.update({utt: self.token_limit_error for utt, _ in files})
        elif files:
            errors.update(self._decode(files))
        for _, em in files:
            em.close()
        each = (time.perf_counter() - t0) / max(len(group), 1)
        for utt, _ in group:
            self.seconds[utt] = each
            if utt in errors:
                log.error("utterance %s failed: %s", utt, errors[utt])
                self.failed.append(utt)

    def _decode(self, files: list) -> dict:
        from . import _lib

        torch, dec = self.torch, self.dec
        V, B = len(self.tokens), len(files)
        T = max(max(em.frames for _, em in files), 1)
        host = torch.zeros((B, T, V), dtype=torch.float32, pin_memory=True)
        staged = host.numpy()
        lens = np.array([em.frames for _, em in files], dtype=np.int32)
        for b, (_, em) in enumerate(files):
            em.copy_to(staged[b])
        x = host.to(dec.device, non_blocking=True)
        lens_dev = torch.from_numpy(lens).to(dec.device)
        errors = {}
        # EmissionMatrix checks (emissions.py:128-150) run inside the decode
        # (ctcb_set_validate): every invalid utterance comes back with its own
        # status and first offender
        dec.set_validate("strict" if self.strict else "nonstrict")
        out = dec.decode(x, lens_dev, timesteps=True)
        status = out.status.cpu().numpy()
        counts = out.counts.cpu().numpy()
        lengths = out.lengths.cpu().numpy()
        scores = out.scores.cpu().numpy()
        width = int(lengths.max()) if lengths.size else 0
        tok = out.tokens[:, :, :width].cpu().numpy()
        ts = out.timesteps[:, :, :width].cpu().numpy()
        lms = out.lm.cpu().numpy() if out.lm is not None else None
        for b, (utt, _) in enumerate(files):
            if status[b] in (_lib.UTT_NONFINITE, _lib.UTT_ABOVE_ZERO, _lib.UTT_NOT_NORMALIZED):
                errors[utt] = _validation_message(int(status[b]) - 4, staged[b].astype(np.float64),
                                                  int(lengths[b, 0]), int(counts[b]))
                continue
            if status[b] == _lib.UTT_EMPTY:
                errors[utt] = "empty emissions"  # decoder.py:117-118
                continue
            if status[b] == _lib.UTT_BEAM_DIED:
                limit = dec.beam_size_token or V
                errors[utt] = (f"beam died at frame {int(lengths[b, 0])}: no extension survives "
                               f"(beam_size_token={limit} may be too small)")
                continue
            hyps = []
            for r in range(int(counts[b])):
                ids = tok[b, r, : lengths[b, r]].tolist()
                hyps.append(self._hypothesis(r, ids, float(scores[b, r]),
                                             float(lms[b, r]) if lms is not None else None,
                                             ts[b, r, : lengths[b, r]].tolist()))
            self.records.append({"utt": utt, "nbest": hyps})
        return errors

    def _hypothesis(self, rank: int, ids: list, score: float, lm_total, timesteps: list) -> dict:
        # am_score = score - lm_weight * lm - silence bonuses (decoder.py:805-812;
        # word_score is lexicon-only)
        sil = self.tokens.silence_index
        bonus = self.opts.sil_score * (ids.count(sil) if sil is not None else 0)
        lm_v = lm_total if lm_total is not None else 0.0
        am = score - (self.opts.lm_weight * lm_v if lm_total is not None else 0.0) - bonus
        names = self.tokens.tokens
        return {"rank": rank, "score": score, "am_score": am, "lm_score": lm_v, "token_ids": ids,
                "tokens": [names[i] for i in ids], "words": [], "timesteps": timesteps}

    def finish(self, out_path: str) -> int:
        self.records.sort(key=lambda r: r["utt"])
        with open(out_path, "w", encoding="utf-8") as fh:
            fh.writelines(_record_line(r) for r in self.records)
        meta = {"command": "decode", "total_time_s": sum(self.seconds.values()),
                "utterances": dict(sorted(self.seconds.items())), "failed": sorted(self.failed),
                "options": dataclasses.asdict(self.opts)}
        Path(out_path + ".meta").write_text(json.dumps(meta, sort_keys=True, indent=2) + "\n", encoding="utf-8")
        log.info("decoded %d utterances (%d failed)", len(self.records), len(self.failed))
        return 1 if self.failed else 0


def _validation_message(code: int, lp: np.ndarray, t: int, v: int) -> str:
    """Validation check code -> EmissionMatrix's message (emissions.py:133-150)."""
    if code == 1:
        return f"non-finite log-probability at frame {t}, token {v}"
    if code == 2:
        return f"log-probability above 0 at frame {t}, token {v}: {lp[t, v]:.6g}"
    m = lp[t].max()
    lse = m + np.log(np.exp(lp[t] - m).sum())
    return (f"frame {t} is not normalized: log-sum-exp = {lse:.6g} (tolerance {ROW_NORM_TOL}); "
            "pass strict=False to skip this check")


# =========================================================================== align
def cmd_align(cfg: dict) -> int:
    """Force-align transcripts (cli.py:327-388): one ``ctcb_align`` launch per
    batch of utterances, records in utterance order, an ``{"utt", "error"}``
    record for each failed utterance."""
    _require(cfg, "emissions", "tokens", "refs")
    _must_exist(cfg, "emissions", "tokens", "refs", "lexicon")
    tokens = _token_dictionary(cfg)
    lexicon = parse_lexicon(cfg["lexicon"], tokens) if cfg["lexicon"] else None
    refs = read_refs(cfg["refs"])
    utts = _utterances(cfg["emissions"])
    from . import align as galign

    aligner = _Aligner(cfg, tokens, lexicon, refs, galign)
    out = sys.stdout if cfg["out"] is None else open(cfg["out"], "w", encoding="utf-8")
    try:
        per_launch = int(cfg["gpu_batch"])
        for k in range(0, len(utts), per_launch):
            out.writelines(aligner.run_batch(utts[k: k + per_launch]))
    finally:
        if out is not sys.stdout:
            out.close()
    return 1 if aligner.failed else 0


class _Aligner:
    def __init__(self, cfg: dict, tokens: TokenDictionary, lexicon, refs: dict, galign):
        self.cfg, self.tokens, self.lexicon, self.refs, self.galign = cfg, tokens, lexicon, refs, galign
        self.index = {t: i for i, t in enumerate(tokens.tokens)}
        self.failed = 0

    def _targets(self, transcript: list) -> list:
        if self.lexicon is None:  # TokenDictionary.index (emissions.py:69-73): a KeyError
            unknown = next((t for t in transcript if t not in self.index), None)
            if unknown is not None:
                raise KeyError(f"unknown token: {unknown!r}")
            return [self.index[t] for t in transcript]
        spelled = []
        for word in transcript:
            variants = self.lexicon.entries.get(word)
            if not variants:
                raise ValueError(f"word {word!r} is not in the lexicon")
            spelled += variants[0]
        return spelled

    def _prepare(self, utt: str, path: Path):
        if utt not in self.refs:
            raise ValueError(f"no transcript for {utt} in --refs")
        lp = parse_emissions(path, len(self.tokens))
        check_emission_matrix(lp, bool(self.cfg["strict_validation"]))
        return self.refs[utt], lp, self._targets(self.refs[utt])

    def run_batch(self, group: list) -> list:
        outcome, ready = {}, []
        for utt, path in group:
            try:
                ready.append((utt, *self._prepare(utt, path)))
            except Exception as exc:  # noqa: BLE001 - per-utterance failure (cli.py:339-344)
                outcome[utt] = exc
        if ready:
            results = self.galign.forced_align_batch([r[2] for r in ready], [r[3] for r in ready], self.tokens,
                                                     device=_device_index(self.cfg["device"]), raise_errors=False)
            for (utt, transcript, _, _), res in zip(ready, results):
                outcome[utt] = ValueError(res) if isinstance(res, str) else (transcript, res)
        lines = []
        for utt, _ in group:
            try:
                got = outcome[utt]
                if isinstance(got, Exception):
                    raise got
                lines += [_record_line(r) for r in self._records(utt, *got)]
            except Exception as exc:  # noqa: BLE001
                lines.append(_record_line({"utt": utt, "error": str(exc)}))
                log.error("utterance %s failed: %s", utt, exc)
                self.failed += 1
        return lines

    def _records(self, utt: str, transcript: list, result) -> list:
        galign = self.galign
        spans = galign.attribute_blanks(result) if self.cfg["attribute_blanks"] else result.spans
        recs = [dict(utt=utt, token=self.tokens.tokens[s.token], start=s.start_frame, end=s.end_frame,
                     score=s.score, prob=math.exp(s.score)) for s in spans]
        if self.lexicon is not None:
            recs += [dict(utt=utt, word=w.word, start=w.start_frame, end=w.end_frame, score=w.score,
                          prob=math.exp(w.score))
                     for w in galign.align_words(result, self.tokens, transcript, self.lexicon)]
        return recs


# =========================================================================== command line
def _flags(p: argparse.ArgumentParser, *names: str) -> None:
    """Shared flags; every default is _UNSET so only given flags override
    the config file."""
    spec = {
        "config": dict(help="JSON config file"),
        "tokens": dict(help="token file, one token per line"),
        "blank-token": dict(), "silence-token": dict(),
        "strict-validation": dict(action=argparse.BooleanOptionalAction),
        "emissions": dict(help="emission file or directory"),
        "gpu-batch": dict(type=int, help="utterances per launch"),
        "device": dict(help="CUDA device: N, cuda or cuda:N"),
        "lexicon": dict(), "lm": dict(),
        "beam-size": dict(type=int), "beam-size-token": dict(type=int), "beam-threshold": dict(type=float),
        "lm-weight": dict(type=float), "word-score": dict(type=float), "sil-score": dict(type=float),
        "blank-skip-threshold": dict(type=float,
                                     help="drop frames with at least this blank probability (1.0 disables)"),
        "nbest": dict(type=int), "merge": dict(choices=["max", "logadd"]),
        "workers": dict(type=int, help="accepted for compatibility (the GPU batches)"),
        "refs": dict(help="transcripts: utt_id<TAB>words"),
        "attribute-blanks": dict(action=argparse.BooleanOptionalAction,
                                 help="widen spans so blanks attach to the preceding token"),
    }
    for name in names:
        p.add_argument(f"--{name}", dest=name.replace("-", "_"), default=_UNSET, **spec.get(name, {}))


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="paper_2310_17864_b200",
                                     description="CTC beam-search decoding on the GPU (ctcforge decode)")
    sub = parser.add_subparsers(dest="command", required=True)
    dec = sub.add_parser("decode", help="beam-search decode emission files")
    _flags(dec, "config", "tokens", "blank-token", "silence-token", "strict-validation", "lexicon", "lm",
           "beam-size", "beam-size-token", "beam-threshold", "lm-weight", "word-score", "sil-score",
           "blank-skip-threshold", "nbest", "merge", "emissions")
    dec.add_argument("--out", default=_UNSET, help="output JSON-lines path (required)")
    _flags(dec, "workers", "gpu-batch", "device")
    ali = sub.add_parser("align", help="force-align transcripts to emissions")
    _flags(ali, "config", "tokens", "blank-token", "silence-token", "strict-validation", "emissions", "refs")
    ali.add_argument("--lexicon", default=_UNSET, help="word mode: spell transcript words through this lexicon")
    ali.add_argument("--out", default=_UNSET, help="output JSON-lines path (default: stdout)")
    _flags(ali, "attribute-blanks", "gpu-batch", "device")
    return parser


def main(argv=None) -> int:
    wanted = os.environ.get("CTCFORGE_LOG", "WARNING").upper()
    logging.basicConfig(level=wanted if isinstance(logging.getLevelName(wanted), int) else "WARNING",
                        format="%(levelname)s %(name)s: %(message)s")
    args = build_parser().parse_args(argv)
    command = {"decode": cmd_decode, "align": cmd_align}[args.command]
    try:
        return command(resolve_settings(args))
    except ConfigError as exc:
        print(f"ctcforge {args.command}: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
