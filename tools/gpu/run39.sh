timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r39_bench.json 2> gpurun_out/r39_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --workload c4 --steps 20 --warmup 3 > gpurun_out/r39_bench_c4.json 2>&1; echo "c4 rc=$?"
timeout 300 python tools/ncu_c4tc.py > gpurun_out/r39_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:small_solve_tc -c 1 -o gpurun_out/r39_c4tc python tools/ncu_c4tc.py > gpurun_out/r39_ncu.log 2>&1; echo "ncu rc=$?"
