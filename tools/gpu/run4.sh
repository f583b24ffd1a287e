timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "int8" > gpurun_out/r4_i8.log 2>&1; echo "i8 tests rc=$?"
tail -30 gpurun_out/r4_i8.log
timeout 600 python tools/prec_time.py c5 0,3
timeout 300 python tools/prec_time.py c2 0,3
