python -m paper_1207_1114_b200.build > /dev/null 2>&1
timeout 300 python tools/prec_time.py c5 3 | tail -1
FASTPFP_LIB=varlib/notma.so timeout 300 python tools/prec_time.py c5 3 | tail -1
FASTPFP_LIB=varlib/nomma.so timeout 300 python tools/prec_time.py c5 3 | tail -1
