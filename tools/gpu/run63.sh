timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r63_bench.json 2> gpurun_out/r63_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --workload c4 --steps 20 --warmup 3 > gpurun_out/r63_bench_c4.json 2> gpurun_out/r63_bench_c4.err; echo "c4 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r63_launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/r63_ncu.log 2>&1; echo "ncu rc=$?"
