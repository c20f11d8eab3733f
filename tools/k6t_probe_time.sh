# ncu gpu__time_duration of the K6T passes (config-5 shape, n = 131072) for A/B libraries built with
# tools/build_variant.py, e.g.
#   python tools/build_variant.py k6t_p0 precond_multi.cu
#   python tools/build_variant.py k6t_p1 precond_multi.cu -DK6T_PROBE=1     # no DMMA
#   python tools/build_variant.py k6t_p2 precond_multi.cu -DK6T_PROBE=2     # copy pipeline only
#   K6T_VARIANTS="p0 p1 p2" bash tools/k6t_probe_time.sh
for v in ${K6T_VARIANTS:-p0 p1 p2}; do
KRR_B200_LIB=_variants/libkrr_k6t_$v.so ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k6t" --csv --log-file gpurun_out/s4_k6t_$v.csv python tools/build_profile.py 5 131072 3 > /dev/null 2>&1
python - <<EOF
import csv,collections
rows=list(csv.reader(l for l in open("gpurun_out/s4_k6t_$v.csv") if l.startswith("\"")))
h=rows[0]; ik=h.index("Kernel Name"); iv=h.index("Metric Value")
t=collections.defaultdict(list)
for r in rows[1:]: t[r[ik][16:36]].append(float(r[iv].replace(",",""))/1e6)
print("$v", {k:[round(x,3) for x in v] for k,v in t.items()})
EOF
done
