"""Phase medians of K1-I8 per-tile traces (the output of tools/i8_trace.py).

python tools/i8_trace_stats.py trace.log ...

All times in SM clocks, medians over the first 38 tiles of CTA 0:
  period    tensor-core group-6 start to the next tile's
  mma       group-6 start to group 0 complete (as seen by the epilogue)
  tail      group 0 complete to the end of the last drain stage
  cdw       wait for the tile's column data
  exp       the exp element loop
  colsum    the column-sum transposes
  handoff   end of the element loop to the next tile's first MMA group
"""
import sys

import numpy as np


def stats(path):
    rows = []
    for line in open(path):
        p = line.split()
        if p and p[0].isdigit():
            rows.append([int(x) for x in p[1:17]] + [int(p[17].split("=")[1])])
    a = np.array(rows[:38], dtype=float)
    start = np.concatenate([[0], np.cumsum(a[:-1, 16])])
    g6, g0d, st0 = start + a[:, 10], start + a[:, 15], start + a[:, 4]
    cd, elem, col = start + a[:, 5], start + a[:, 13], start + a[:, 14]
    m = lambda x: float(np.median(x))  # noqa: E731
    return {"period": m(np.diff(g6)), "mma": m(g0d - g6), "tail": m(st0 - g0d), "cdw": m(cd - st0),
            "exp": m(elem - cd), "colsum": m(col - elem), "handoff": m(g6[1:] - elem[:-1]),
            "g6_to_g4_issue": m(a[:, 11] - a[:, 10]), "g4_to_g0_issue": m(a[:, 12] - a[:, 11]),
            "g0_issue_to_done": m(a[:, 15] - a[:, 12])}


if __name__ == "__main__":
    for f in sys.argv[1:]:
        print(f.split("/")[-1], " ".join(f"{k} {v:.0f}" for k, v in stats(f).items()))
