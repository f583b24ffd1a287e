timeout 300 python tools/prec_time.py c5 3 | tail -1
FASTPFP_LIB=varlib/nostore.so timeout 300 python tools/prec_time.py c5 3 | tail -1
FASTPFP_LIB=varlib/nostore2.so timeout 300 python tools/prec_time.py c5 3 | tail -1
