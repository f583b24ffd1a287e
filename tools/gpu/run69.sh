FASTPFP_LIB=varlib/ocprof.so timeout 300 python tools/c2_probe.py 2>&1 | grep -E "oc-prof|pk" | tail -6
