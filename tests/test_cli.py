"""The GPU ``decode`` command (paper_2310_17864_b200/cli.py) against the reference
``ctcforge decode`` (cli.py:262-312): host-side parsing and configuration on the
CPU, full runs on the GPU compared with the reference command's own output on
the golden corpus (tests/golden/make_cli_golden.py)."""

import json
import os
import struct

import numpy as np
import pytest

from paper_2310_17864_b200 import cli

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cli")
CORPUS = os.path.join(GOLD, "corpus")
TOKENS = os.path.join(GOLD, "tokens.txt")


def expected():
    with open(os.path.join(GOLD, "expected.json"), encoding="utf-8") as fh:
        return json.load(fh)


# ------------------------------------------------------------------ CPU: host logic
def test_token_file_rules(tmp_path):
    # emissions.py:79-113: whole stripped line, blank "<blank>" then "-", or --blank-token
    p = tmp_path / "t.txt"
    p.write_text("a\n-\n <blank> \nb\n", encoding="utf-8")
    td = cli.TokenDictionary.from_file(p)
    assert td.tokens == ("a", "-", "<blank>", "b") and td.blank_index == 2
    assert cli.TokenDictionary.from_file(p, blank_token="a").blank_index == 0
    assert cli.TokenDictionary.from_file(p, silence_token="b").silence_index == 3
    with pytest.raises(ValueError, match="no blank token found"):
        cli.TokenDictionary.from_file(p, blank_token="zz")
    with pytest.raises(ValueError, match="silence token 'zz' not in token file"):
        cli.TokenDictionary.from_file(p, silence_token="zz")
    p.write_text("a\n\n-\n", encoding="utf-8")
    with pytest.raises(ValueError, match="line 2: empty token"):
        cli.TokenDictionary.from_file(p)
    p.write_text("-\na\na\n", encoding="utf-8")
    with pytest.raises(ValueError, match="unique"):
        cli.TokenDictionary.from_file(p)


def test_emission_readers(tmp_path):
    rng = np.random.default_rng(0)
    lp = np.log(rng.dirichlet(np.ones(5), size=7)).astype(np.float32)
    cli.write_emissions(lp, tmp_path / "a.ctce")
    assert np.array_equal(cli.parse_emissions(tmp_path / "a.ctce", 5), lp)
    (tmp_path / "b.tsv").write_text("\n".join("\t".join(repr(float(x)) for x in r) for r in lp) + "\n")
    assert np.array_equal(cli.parse_emissions(tmp_path / "b.tsv", 5), lp)
    with pytest.raises(ValueError, match="5 columns but the token dictionary has 6 tokens"):
        cli.parse_emissions(tmp_path / "a.ctce", 6)
    raw = (tmp_path / "a.ctce").read_bytes()
    (tmp_path / "c.ctce").write_bytes(raw[:-4])
    with pytest.raises(ValueError, match="expected 156 bytes for a 7x5 matrix, got 152"):
        cli.parse_emissions(tmp_path / "c.ctce", 5)
    (tmp_path / "d.ctce").write_bytes(struct.pack("<4sIII", b"CTCE", 2, 1, 5) + bytes(20))
    with pytest.raises(ValueError, match="unsupported version 2"):
        cli.parse_emissions(tmp_path / "d.ctce", 5)
    (tmp_path / "e.tsv").write_text("0\t-1\nnan\t0\n")
    with pytest.raises(ValueError, match="non-finite value at frame 1, column 0"):
        cli.parse_emissions(tmp_path / "e.tsv", 2)
    (tmp_path / "f.tsv").write_text("0\t-1\n0\n")
    with pytest.raises(ValueError, match="line 2: expected 2 columns, got 1"):
        cli.parse_emissions(tmp_path / "f.tsv", 2)
    (tmp_path / "g.ctce").write_bytes(b"CTC")  # short, sniffed as TSV (as the reference does)
    with pytest.raises(ValueError, match="line 1: could not convert string to float"):
        cli.parse_emissions(tmp_path / "g.ctce", 2)
    (tmp_path / "h.bin").write_bytes(b"\xff\xfe\x00")
    with pytest.raises(ValueError, match="neither CTCE binary nor UTF-8 TSV"):
        cli.parse_emissions(tmp_path / "h.bin", 2)


def test_config_errors_exit_2(tmp_path, capsys):
    out = str(tmp_path / "o.jsonl")
    base = ["decode", "--emissions", CORPUS, "--tokens", TOKENS]
    assert cli.main(base) == 2 and "--out is required" in capsys.readouterr().err
    assert cli.main(base + ["--out", out, "--lm", str(tmp_path / "missing.arpa")]) == 2
    assert "file not found" in capsys.readouterr().err
    lm = tmp_path / "x.arpa"
    lm.write_text("\\data\\\n")
    assert cli.main(base + ["--out", out, "--lm", str(lm)]) == 2 and "ngram N=count" in capsys.readouterr().err
    assert cli.main(base + ["--out", out, "--lexicon", str(lm)]) == 2 and "lexicon-free" in capsys.readouterr().err
    assert cli.main(base + ["--out", out, "--nbest", "20"]) == 2 and "n_best" in capsys.readouterr().err
    cfg = tmp_path / "c.json"
    cfg.write_text(json.dumps({"bogus": 1}))
    assert cli.main(base + ["--out", out, "--config", str(cfg)]) == 2 and "unknown key" in capsys.readouterr().err


def test_device_argument():
    assert cli._device_index("cuda") == 0 and cli._device_index("cuda:3") == 3 and cli._device_index(2) == 2
    with pytest.raises(cli.ConfigError, match="--device"):
        cli._device_index("cpu")


def test_config_precedence(tmp_path):
    # CLI > --config file > defaults (cli.py:130-148)
    cfg = tmp_path / "c.json"
    cfg.write_text(json.dumps({"beam_size": 7, "nbest": 2, "merge": "max"}))
    args = cli.build_parser().parse_args(["decode", "--config", str(cfg), "--nbest", "3"])
    merged = cli.resolve_settings(args)
    assert merged["beam_size"] == 7 and merged["nbest"] == 3 and merged["merge"] == "max"
    assert merged["beam_threshold"] == 50.0


# ------------------------------------------------------------------ GPU: full command
@pytest.mark.gpu
@pytest.mark.parametrize("run", ["default", "beam5_nbest3_skip", "max_merge", "nonstrict", "lm_bigram",
                                 "lm_silence"])
def test_decode_matches_reference_command(tmp_path, run):
    exp = expected()[run]
    out = str(tmp_path / "o.jsonl")
    flags = [os.path.join(GOLD, f) if f.endswith(".arpa") else f for f in exp["flags"]]
    rc = cli.main(["decode", "--emissions", CORPUS, "--tokens", TOKENS, "--out", out] + flags)
    assert rc == exp["exit_code"]
    with open(out, encoding="utf-8") as fh:
        got = [json.loads(line) for line in fh]
    with open(out + ".meta", encoding="utf-8") as fh:
        meta = json.load(fh)
    assert meta["failed"] == exp["failed"]
    assert meta["options"] == exp["options"]
    assert [r["utt"] for r in got] == [r["utt"] for r in exp["records"]]
    for g, e in zip(got, exp["records"]):
        assert len(g["nbest"]) == len(e["nbest"]), g["utt"]
        for a, b in zip(g["nbest"], e["nbest"]):
            for key in ("rank", "token_ids", "tokens", "words", "timesteps"):
                assert a[key] == b[key], (g["utt"], key)
            assert a["lm_score"] == pytest.approx(b["lm_score"], abs=1e-9)
            assert a["score"] == pytest.approx(b["score"], abs=1e-9)
            assert a["am_score"] == pytest.approx(b["am_score"], abs=1e-9)


@pytest.mark.gpu
def test_decode_single_file_and_small_batches(tmp_path):
    exp = expected()["default"]
    out = str(tmp_path / "o.jsonl")
    # batches of 3 utterances per launch give the same records
    assert cli.main(["decode", "--emissions", CORPUS, "--tokens", TOKENS, "--out", out, "--gpu-batch", "3"]) == 1
    with open(out, encoding="utf-8") as fh:
        assert [json.loads(line)["utt"] for line in fh] == [r["utt"] for r in exp["records"]]
    assert cli.main(["decode", "--emissions", os.path.join(CORPUS, "utt03.ctce"), "--tokens", TOKENS,
                     "--out", out]) == 0
    with open(out, encoding="utf-8") as fh:
        rec = [json.loads(line) for line in fh]
    ref = [r for r in exp["records"] if r["utt"] == "utt03"]
    assert [r["nbest"][0]["token_ids"] for r in rec] == [r["nbest"][0]["token_ids"] for r in ref]


def _norm_paths(records):
    # error texts carry the emission file path of the machine that ran the command
    out = []
    for r in records:
        r = dict(r)
        if "error" in r:
            r["error"] = r["error"].replace(os.path.abspath(CORPUS) + os.sep, "").replace(
                "/root/repo/tests/golden/cli/corpus/", "")
        out.append(r)
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("run", ["align_tokens", "align_tokens_tiled", "align_tokens_nonstrict", "align_words"])
def test_align_matches_reference_command(tmp_path, run):
    """The GPU align command (token and word modes, tiled spans, per-utterance
    error records) against the reference `ctcforge align` output."""
    exp = expected()[run]
    flags = [os.path.join(GOLD, f) if f.endswith(".txt") else f for f in exp["flags"]]
    out = str(tmp_path / "a.jsonl")
    rc = cli.main(["align", "--emissions", CORPUS, "--tokens", TOKENS, "--out", out] + flags)
    assert rc == exp["exit_code"]
    with open(out, encoding="utf-8") as fh:
        got = [json.loads(line) for line in fh]
    assert _norm_paths(got) == _norm_paths(exp["records"])
