# ncu --set full of the config-5 Woodbury build's K5 TRSM (one mid-build column block) and of the
# 16-column K6T apply (pass a + pass b), via tools/build_profile.py.  Run alone on one GPU (gpurun).
set -e
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:trsm_block --launch-skip 64 -c 1 \
    -o gpurun_out/trsm_c5 python tools/build_profile.py 5 524288 1 > gpurun_out/ncu_trsm_c5.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k6t_pass -c 2 \
    -o gpurun_out/k6t_c5 python tools/build_profile.py 5 524288 1 > gpurun_out/ncu_k6t_c5.log 2>&1
