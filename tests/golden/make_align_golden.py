"""Golden vectors for CTC forced alignment from the REFERENCE
(ctcforge.align.forced_align, /root/reference/pkg/src/ctcforge/align.py:46-139),
imported in the build container (it does not exist on the GPU box):

    python tests/golden/make_align_golden.py

Writes ``tests/golden/align.json``: float32-exact emissions (so the float32
CUDA path sees the reference's exact inputs), targets, and the reference's
frame labels, frame scores and token spans -- or its error message.  Cases:
peaked / flat / uniform (all ties) rows, adjacent repeats, the feasibility
boundary T = L + repeats, single-token targets, and the argument errors.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from ctcforge.align import attribute_blanks, forced_align  # noqa: E402
from ctcforge.emissions import EmissionMatrix, TokenDictionary  # noqa: E402


def logsoftmax32(x):
    x = x - x.max(1, keepdims=True)
    return (x - np.log(np.exp(x).sum(1, keepdims=True))).astype(np.float32)


def main():
    rng = np.random.default_rng(20261019)
    cases = []

    def add(lp32, targets, blank=0, note=""):
        V = lp32.shape[1]
        tokens = TokenDictionary(tuple(["<b>"] + [f"t{i}" for i in range(1, V)]), blank_index=blank) if blank == 0 \
            else TokenDictionary(tuple(f"t{i}" for i in range(V)), blank_index=blank)
        em = EmissionMatrix(lp32.astype(np.float64), strict=False)
        case = {"note": note, "lp": lp32.astype(np.float64).tolist(), "targets": [int(t) for t in targets],
                "blank": blank}
        try:
            r = forced_align(em, targets, tokens)
            case["labels"] = r.frame_labels.tolist()
            case["scores"] = r.frame_scores.tolist()
            case["spans"] = [[s.token, s.start_frame, s.end_frame, s.score] for s in r.spans]
            case["tiled"] = [[s.token, s.start_frame, s.end_frame, s.score] for s in attribute_blanks(r)]
        except ValueError as exc:
            case["error"] = str(exc)
        cases.append(case)

    for i in range(40):  # random peaky utterances
        V = int(rng.integers(4, 40))
        T = int(rng.integers(3, 60))
        L = int(rng.integers(1, max(2, T // 2)))
        targets = rng.integers(1, V, size=L)
        if i % 4 == 0 and L > 1:
            targets[1] = targets[0]  # adjacent repeat
        logits = rng.normal(0, 1.0, size=(T, V))
        for t in range(T):
            if rng.random() < 0.5:
                logits[t, 0] += rng.uniform(2, 6)
            else:
                logits[t, targets[min(L - 1, t * L // T)]] += rng.uniform(2, 6)
        add(logsoftmax32(logits), targets, note="random")
    for i in range(10):  # flat rows: many near-ties
        V, T = int(rng.integers(3, 8)), int(rng.integers(4, 30))
        L = int(rng.integers(1, max(2, T // 3)))
        add(logsoftmax32(rng.normal(0, 0.05, size=(T, V))), rng.integers(1, V, size=L), note="flat")
    add(logsoftmax32(np.zeros((6, 4))), [1, 2], note="uniform ties")
    add(logsoftmax32(np.zeros((5, 3))), [1, 1, 2], note="uniform, repeat")
    add(logsoftmax32(rng.normal(0, 1, size=(4, 5))), [2, 2, 3], note="boundary T = L + repeats")
    add(logsoftmax32(rng.normal(0, 1, size=(3, 5))), [2, 2, 3], note="infeasible")
    add(logsoftmax32(rng.normal(0, 1, size=(1, 5))), [3], note="single frame")
    add(logsoftmax32(rng.normal(0, 1, size=(7, 5))), [], note="empty targets")
    add(logsoftmax32(rng.normal(0, 1, size=(7, 5))), [1, 0], note="blank target")
    add(logsoftmax32(rng.normal(0, 1, size=(7, 5))), [1, 9], note="out of range")
    add(logsoftmax32(rng.normal(0, 2, size=(12, 6))), [1, 4], blank=3, note="blank index 3")
    with open(os.path.join(HERE, "align.json"), "w", encoding="utf-8") as fh:
        json.dump({"cases": cases}, fh)
    print(len(cases), "cases;", sum("error" in c for c in cases), "errors")


if __name__ == "__main__":
    main()
