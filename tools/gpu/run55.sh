FASTPFP_LIB=varlib/clk.so timeout 300 python tools/prec_time.py c5 3 > /tmp/a.log 2>&1; grep i8-clk /tmp/a.log | tail -3; tail -1 /tmp/a.log
FASTPFP_LIB=varlib/prof.so timeout 300 python tools/prec_time.py c5 3 > /tmp/a.log 2>&1; grep i8-prof /tmp/a.log | tail -2; tail -1 /tmp/a.log
