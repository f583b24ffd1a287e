for v in "" build/var_skipp/libfastpfp.so; do echo "lib=$v"; FASTPFP_LIB=$v timeout 600 python tools/prec_time.py c5 3 2>&1 | tail -1; done
