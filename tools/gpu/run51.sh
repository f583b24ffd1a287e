timeout 300 python tools/prec_time.py c5 3 | tail -1
FASTPFP_LIB=varlib/notma.so timeout 300 python tools/prec_time.py c5 3 | tail -1
