FASTPFP_LIB=varlib/prof.so timeout 300 python tools/prec_time.py c5 3 > /tmp/a.log 2>&1; grep i8-prof /tmp/a.log | tail -4; tail -1 /tmp/a.log
FASTPFP_LIB=varlib/prof_old.so timeout 300 python tools/prec_time.py c5 3 > /tmp/b.log 2>&1; grep i8-prof /tmp/b.log | tail -4; tail -1 /tmp/b.log
