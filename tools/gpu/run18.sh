timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r18_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r18_tests.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r18_bench.json 2> gpurun_out/r18_bench.err; echo "bench rc=$?"
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-secondary --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/r18_plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r18_launches.csv $CMD > gpurun_out/r18_ncu1.log 2>&1; echo "ncu1 rc=$?"
timeout 600 $CMD > gpurun_out/r18_plain2.log 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on -k regex:gemm_i8 -s 2 -c 1 -o gpurun_out/r18_gemm_i8 $CMD > gpurun_out/r18_ncu2.log 2>&1; echo "ncu2 rc=$?"
timeout 600 $CMD > gpurun_out/r18_plain3.log 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on -k regex:proj_kernel -s 1 -c 1 -o gpurun_out/r18_proj $CMD > gpurun_out/r18_ncu3.log 2>&1; echo "ncu3 rc=$?"
