for v in "" build/var_t384/libfastpfp.so build/var_t512/libfastpfp.so; do echo "lib=$v"; FASTPFP_LIB=$v timeout 300 python tools/c2_probe.py 2>&1 | tail -3; done
