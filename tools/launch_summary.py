"""Per-kernel totals of an ncu launch list (`ncu --metrics gpu__time_duration.sum --csv --log-file F`).

python tools/launch_summary.py F.csv "comment line"
"""
import collections
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hdr, tot, cnt = None, collections.defaultdict(float), collections.Counter()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] != "gpu__time_duration.sum":
                continue
            name = d["Kernel Name"].split("(")[0].replace("krr::<", "").replace("(anonymous namespace)::", "")
            v = float(d["Metric Value"].replace(",", ""))
            unit = d.get("Metric Unit", "ns")
            ms = v * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "msecond": 1.0, "ms": 1.0, "nsecond": 1e-6}.get(unit, 1e-6)
            tot[name] += ms
            cnt[name] += 1
    all_ms = sum(tot.values())
    if len(sys.argv) > 2:
        print("# " + sys.argv[2])
    print(f"# total GPU time of the captured launches: {all_ms:.1f} ms")
    print("# kernel  launches  total_ms  share")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{k[-64:]:64s} {cnt[k]:4d} {v:12.3f} {100 * v / all_ms:6.2f}%")


if __name__ == "__main__":
    main()
