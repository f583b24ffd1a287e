./tools/micro/gridsync
FASTPFP_LIB=build/var_ocprof/libfastpfp.so timeout 300 python tools/c2_probe.py 2>&1 | tail -12
