FASTPFP_LIB=varlib/ssprof.so timeout 300 python tools/c4_split.py 2>&1 | grep -E "ss-prof|c4 20" | tail -4
timeout 300 python tools/c4_split.py 2>&1 | tail -3
