timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r68_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r68_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r68_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r68_bench.json 2> gpurun_out/r68_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --workload c4 --steps 20 --warmup 3 > gpurun_out/r68_bench_c4.json 2> gpurun_out/r68_bench_c4.err; echo "c4 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r68_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-secondary --no-cpu-baseline > gpurun_out/r68_ncu.log 2>&1; echo "ncu rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_i8 -s 2 -c 1 -o gpurun_out/r68_gemm python tools/prec_time.py c5 3 > gpurun_out/r68_ncu_gemm.log 2>&1; echo "ncu gemm rc=$?"
