for v in "" build/var_relax/libfastpfp.so build/var_relax_u4/libfastpfp.so build/var_u4/libfastpfp.so; do echo "lib=$v"; FASTPFP_LIB=$v timeout 300 python tools/c2_probe.py 2>&1 | grep "pk 0"; done
