for i in 1 2; do
timeout 300 python tools/prec_time.py c5 3 | tail -1
FASTPFP_LIB=varlib/hint.so timeout 300 python tools/prec_time.py c5 3 2>&1 | tail -1
FASTPFP_LIB=varlib/dp.so timeout 300 python tools/prec_time.py c5 3 2>&1 | tail -1
done
