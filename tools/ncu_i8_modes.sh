# ncu --set full of one K1-I8 launch (n = 65536, d = 90) with the MMAs off (i8_debug 1) and on.
# The profiling modes need a build with -DI8_PROFILE=1 (tools/build_variant.py prof gauss_matvec_i8.cu -DI8_PROFILE=1
# and KRR_B200_LIB=_variants/libkrr_prof.so); the default lean build ignores i8_debug bits 1, 2, 16, 32.
set -e
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gauss_matvec_i8 -c 1 -o gpurun_out/i8_nomma python tools/one_i8_launch.py 1 > gpurun_out/ncu_nomma.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gauss_matvec_i8 -c 1 -o gpurun_out/i8_full python tools/one_i8_launch.py 0 > gpurun_out/ncu_full.log 2>&1
