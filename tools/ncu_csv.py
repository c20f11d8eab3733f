"""Print kernel / metric / value rows of an `ncu --csv --log-file` metrics capture.
  python tools/ncu_csv.py FILE.csv [name-substring]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
flt = sys.argv[2] if len(sys.argv) > 2 else ""
hdr = None
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if flt in d["Kernel Name"]:
            print(f'{d["ID"]:>4} {d["Kernel Name"].split("(")[0][-44:]:44s} {d["Metric Name"]:52s} {d["Metric Value"]}')
