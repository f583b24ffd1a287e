for v in "" build/var_kb64/libfastpfp.so build/var_kb64s3/libfastpfp.so; do echo "lib=$v"; FASTPFP_LIB=$v timeout 600 python tools/prec_time.py c5 3 2>&1 | tail -1; done
FASTPFP_LIB=build/var_kb64/libfastpfp.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "int8 and (gemm or config2 or config5)" 2>&1 | tail -2
