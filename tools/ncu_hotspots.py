"""Summarise an ncu report of K1: key metrics + SASS-level warp-stall hot spots.

python tools/ncu_hotspots.py gpurun_out/k1_d90.ncu-rep [--top 30]
"""
import argparse
import collections
import csv
import io
import subprocess

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "launch__registers_per_thread", "launch__grid_size"]


def ncu(args):
    return subprocess.run(["ncu"] + args, capture_output=True, text=True).stdout


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--top", type=int, default=30)
    a = ap.parse_args()
    raw = list(csv.reader(io.StringIO(ncu(["-i", a.rep, "--page", "raw", "--csv"]))))
    hdr, units, vals = raw[0], raw[1], raw[2]
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))
    for k in KEYS:
        if k in d:
            print(f"{k:85s} {d[k]:>18s} {u.get(k, '')}")
    stalls = {k: float(v) for k, v in d.items()
              if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")
              and v not in ("", "n/a")}
    print("stalls (warps per issue):",
          ", ".join(f"{k[34:-23]}={v:.2f}" for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:8]))

    src = ncu(["-i", a.rep, "--page", "source", "--csv", "--print-source", "sass"])
    lines = src.splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
    rows = list(csv.reader(lines[start:]))
    h = rows[0]
    isrc, isamp = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
    data = rows[1:]
    samp = [float(r[isamp] or 0) for r in data]
    tot = sum(samp) or 1.0
    ops = [r[isrc].strip() for r in data]
    dmma = [i for i, o in enumerate(ops) if "DMMA" in o]
    lo, hi = (dmma[0] - 30, dmma[-1] + 2) if dmma else (0, -1)
    main_share = sum(samp[lo:hi + 1]) / tot
    print(f"samples {tot:.0f}; mainloop region [{lo},{hi}] {100 * main_share:.1f}%; rest {100 * (1 - main_share):.1f}%")
    by = collections.Counter()
    for o, s in zip(ops, samp):
        w = o.split()
        op = (w[1] if w and w[0].startswith("@") and len(w) > 1 else (w[0] if w else "")).split(".")[0]
        by[op] += s
    print("by opcode:", ", ".join(f"{k}={100 * v / tot:.1f}%" for k, v in by.most_common(14)))
    top = sorted(range(len(data)), key=lambda i: -samp[i])[: a.top]
    for i in sorted(top):
        print(f"{i:5d} {100 * samp[i] / tot:5.2f}%  {ops[i][:90]}")


if __name__ == "__main__":
    main()
