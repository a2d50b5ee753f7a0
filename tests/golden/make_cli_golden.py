"""Generate the CLI golden corpus by running the REFERENCE ``ctcforge decode``
command (imported from /root/reference in the build container; it does not exist
on the GPU box):

    python tests/golden/make_cli_golden.py

Writes ``tests/golden/cli/``: ``tokens.txt``, ``corpus/*.ctce|*.tsv`` (seeded
peaky posteriors, float32-exact; plus a wrong-width file and a non-normalized
file that fail per utterance), and for each option set in RUNS the reference's
JSON-lines output, its ``.meta`` failed list and exit code (``expected.json``).
"""

from __future__ import annotations

import json
import os
import shutil
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "cli")
sys.path.insert(0, "/root/reference/pkg/src")

from ctcforge import cli as ref_cli  # noqa: E402
from ctcforge.emissions import EmissionMatrix, write_emissions  # noqa: E402

V = 12
TOKENS = ["<blank>"] + [f"u{i}" for i in range(1, V)]
RUNS = {
    "default": [],
    "beam5_nbest3_skip": ["--beam-size", "5", "--nbest", "3", "--blank-skip-threshold", "0.9"],
    "max_merge": ["--merge", "max", "--beam-size", "8", "--nbest", "2", "--beam-threshold", "6.0"],
    "nonstrict": ["--no-strict-validation", "--beam-size", "4"],
    # token-level LM fusion (lm.arpa: seeded synthetic bigram over the token strings)
    "lm_bigram": ["--lm", "lm.arpa", "--lm-weight", "1.5", "--beam-size", "6", "--nbest", "2"],
    "lm_silence": ["--lm", "lm.arpa", "--lm-weight", "0.8", "--silence-token", "u11", "--sil-score", "0.7",
                   "--nbest", "3", "--blank-skip-threshold", "0.95"],
}


def write_lm(path):
    """Seeded synthetic bigram model over u1..u10 (u11 is out of vocabulary)."""
    rng = np.random.default_rng(7)
    vocab = ["<s>", "</s>"] + TOKENS[1:-1]
    lines = ["\\data\\", f"ngram 1={len(vocab)}", "ngram 2=PLACEHOLDER", "", "\\1-grams:"]
    for w in vocab:
        p = -99.0 if w == "<s>" else rng.uniform(-2.0, -0.4)
        lines.append(f"{p:.4f}\t{w}\t{rng.uniform(-0.7, 0.1):.4f}")
    big = []
    for a in vocab[:1] + vocab[2:]:
        for b in vocab[1:]:
            if rng.random() < 0.4:
                big.append(f"{rng.uniform(-1.8, -0.05):.4f}\t{a} {b}")
    lines += ["", "\\2-grams:"] + big + ["", "\\end\\", ""]
    with open(path, "w", encoding="utf-8") as fh:
        fh.write("\n".join(lines).replace("PLACEHOLDER", str(len(big))))


def utterance(rng, t):
    logits = rng.normal(0.0, 1.0, size=(t, V))
    for i in range(t):
        if rng.random() < 0.55:
            logits[i, 0] += rng.uniform(4, 9)
        else:
            logits[i, rng.integers(1, V)] += rng.uniform(3, 7)
    lp = logits - np.log(np.exp(logits - logits.max(1, keepdims=True)).sum(1, keepdims=True)) - logits.max(1, keepdims=True)
    return lp.astype(np.float32)


def main():
    shutil.rmtree(OUT, ignore_errors=True)
    corpus = os.path.join(OUT, "corpus")
    os.makedirs(corpus)
    with open(os.path.join(OUT, "tokens.txt"), "w", encoding="utf-8") as fh:
        fh.write("\n".join(TOKENS) + "\n")
    rng = np.random.default_rng(20261019)
    for i in range(9):
        lp = utterance(rng, int(rng.integers(8, 48)))
        write_emissions(EmissionMatrix(lp.astype(np.float64)), os.path.join(corpus, f"utt{i:02d}.ctce"))
    lp = utterance(rng, 20)
    with open(os.path.join(corpus, "utt09.tsv"), "w", encoding="utf-8") as fh:
        for row in lp:
            fh.write("\t".join(repr(float(x)) for x in row) + "\n")
    # per-utterance failures: wrong width, and a row that does not normalise
    write_emissions(EmissionMatrix(utterance(rng, 6)[:, :V - 1].astype(np.float64), strict=False),
                    os.path.join(corpus, "bad_width.ctce"))
    lp = utterance(rng, 10)
    lp[3] -= 0.5
    write_emissions(EmissionMatrix(lp.astype(np.float64), strict=False), os.path.join(corpus, "unnormalized.ctce"))
    write_lm(os.path.join(OUT, "lm.arpa"))
    expected = {}
    with tempfile.TemporaryDirectory() as tmp:
        for name, flags in RUNS.items():
            out = os.path.join(tmp, name + ".jsonl")
            full = [os.path.join(OUT, f) if f.endswith(".arpa") else f for f in flags]
            rc = ref_cli.main(["decode", "--emissions", corpus, "--tokens", os.path.join(OUT, "tokens.txt"),
                               "--out", out] + full)
            with open(out, encoding="utf-8") as fh:
                records = [json.loads(line) for line in fh]
            with open(out + ".meta", encoding="utf-8") as fh:
                meta = json.load(fh)
            expected[name] = {"flags": flags, "exit_code": rc, "records": records, "failed": meta["failed"],
                              "options": meta["options"]}
    # align: transcripts = the reference's own best decodes (feasible), in token
    # and word form, plus per-utterance failures (missing transcript, unknown
    # token / word, infeasible length)
    best = {r["utt"]: r["nbest"][0]["tokens"] for r in expected["default"]["records"]}
    tok_lines, word_lines, lex = [], [], {}
    for utt, toks in sorted(best.items()):
        if utt == "utt05":
            continue  # no transcript
        t = list(toks) if toks else ["u1"]
        if utt == "utt06":
            t = t + ["zz"]  # unknown token
        if utt == "utt07":
            t = t * 40  # infeasible
        tok_lines.append(utt + "\t" + " ".join(t))
        # words: consecutive token pairs
        words = []
        for i in range(0, len(toks), 2):
            w = "w" + "_".join(toks[i:i + 2])
            lex.setdefault(w, toks[i:i + 2])
            words.append(w)
        if utt == "utt08":
            words.append("notaword")
        word_lines.append(utt + "\t" + " ".join(words or ["wu1"]))
    lex.setdefault("wu1", ["u1"])
    tok_lines.append("bad_width\tu1")
    tok_lines.append("unnormalized\tu1 u2")
    word_lines.append("unnormalized\twu1")
    with open(os.path.join(OUT, "refs_tokens.txt"), "w", encoding="utf-8") as fh:
        fh.write("\n".join(tok_lines) + "\n")
    with open(os.path.join(OUT, "refs_words.txt"), "w", encoding="utf-8") as fh:
        fh.write("\n".join(word_lines) + "\n")
    with open(os.path.join(OUT, "lexicon.txt"), "w", encoding="utf-8") as fh:
        fh.write("# word spelling\n" + "\n".join(f"{w} {' '.join(sp)}" for w, sp in lex.items()) + "\n")
    ALIGN_RUNS = {
        "align_tokens": ["--refs", os.path.join(OUT, "refs_tokens.txt")],
        "align_tokens_tiled": ["--refs", os.path.join(OUT, "refs_tokens.txt"), "--attribute-blanks"],
        "align_tokens_nonstrict": ["--refs", os.path.join(OUT, "refs_tokens.txt"), "--no-strict-validation"],
        "align_words": ["--refs", os.path.join(OUT, "refs_words.txt"), "--lexicon", os.path.join(OUT, "lexicon.txt")],
    }
    with tempfile.TemporaryDirectory() as tmp:
        for name, flags in ALIGN_RUNS.items():
            out = os.path.join(tmp, name + ".jsonl")
            rc = ref_cli.main(["align", "--emissions", corpus, "--tokens", os.path.join(OUT, "tokens.txt"),
                               "--out", out] + flags)
            with open(out, encoding="utf-8") as fh:
                records = [json.loads(line) for line in fh]
            expected[name] = {"flags": [os.path.basename(f) if os.sep in f else f for f in flags],
                              "exit_code": rc, "records": records}
    with open(os.path.join(OUT, "expected.json"), "w", encoding="utf-8") as fh:
        json.dump(expected, fh, sort_keys=True, indent=1)
    print({k: (v["exit_code"], len(v["records"]), v.get("failed")) for k, v in expected.items()})


if __name__ == "__main__":
    main()
