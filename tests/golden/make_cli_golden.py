#!/usr/bin/env python3
"""Makes tests/golden/cli/: FASTA inputs and the reference CLI's output bytes for them.

Run in the build container (needs oracle/_ref/ref_cli, i.e. the reference sources):
    python tests/golden/make_cli_golden.py
The inputs are seeded; outputs come from the unmodified reference library's
compute_plot + write_tsv/write_pgm/write_dots (oracle/ref_cli.cpp).
"""
import json
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
OUT = os.path.join(HERE, "cli")
REF_CLI = os.path.join(ROOT, "oracle", "_ref", "ref_cli")

CASES = [
    # name, window, step, lcs_only, format, dense, threshold
    ("tsv_align", 20, 3, 0, "tsv", 0, None),
    ("tsv_lcs_thr", 16, 1, 1, "tsv", 0, 13),
    ("tsv_dense", 16, 2, 1, "tsv", 1, 13),
    ("pgm_align", 24, 2, 0, "pgm", 0, None),
    ("pgm_thr", 24, 2, 0, "pgm", 0, 9.5),
    ("dots_align", 20, 1, 0, "dots", 0, 10.5),
]


def fasta(name, seq, width=60):
    lines = [f">{name} synthetic"] + [seq[i:i + width] for i in range(0, len(seq), width)]
    return "\n".join(lines) + "\n"


def main():
    os.makedirs(OUT, exist_ok=True)
    rng = np.random.default_rng(4242)
    x = "".join(rng.choice(list("ACGT"), 170))
    y = x[30:130].lower() + "".join(rng.choice(list("acgt"), 60))   # case folding exercised
    with open(os.path.join(OUT, "x.fa"), "w") as f:
        f.write(fasta("x", x))
    with open(os.path.join(OUT, "y.fa"), "w") as f:
        f.write(fasta("y", y, 50))
    index = []
    for name, w, h, lcs, fmt, dense, thr in CASES:
        args = [REF_CLI, os.path.join(OUT, "x.fa"), os.path.join(OUT, "y.fa"), str(w), str(h), str(lcs), fmt,
                str(dense)] + ([str(thr)] if thr is not None else [])
        out = subprocess.run(args, check=True, capture_output=True).stdout
        with open(os.path.join(OUT, f"{name}.{fmt}"), "wb") as f:
            f.write(out)
        index.append({"name": name, "window": w, "step": h, "lcs_only": lcs, "format": fmt, "dense": dense,
                      "threshold": thr, "file": f"{name}.{fmt}"})
    with open(os.path.join(OUT, "index.json"), "w") as f:
        json.dump({"source": "oracle/ref_cli.cpp (reference compute_plot + io.cpp writers)", "cases": index}, f,
                  indent=1)


if __name__ == "__main__":
    main()
