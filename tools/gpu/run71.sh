for i in 1 2 3; do
timeout 300 python tools/prec_time.py c5 3 | tail -1
FASTPFP_LIB=varlib/nofuse.so timeout 300 python tools/prec_time.py c5 3 | tail -1
done
