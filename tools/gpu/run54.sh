for i in 1 2; do
timeout 300 python tools/prec_time.py c5 3 | tail -1
FASTPFP_LIB=varlib/old.so timeout 300 python tools/prec_time.py c5 3 | tail -1
FASTPFP_LIB=varlib/prof.so timeout 300 python tools/prec_time.py c5 3 2>&1 | tail -1
done
nvidia-smi --query-gpu=power.limit,power.draw,clocks.sm,temperature.gpu --format=csv
