timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r79_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r79_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r79_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r79_bench.json 2> gpurun_out/r79_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --workload c4 --steps 20 --warmup 3 > gpurun_out/r79_bench_c4.json 2> gpurun_out/r79_bench_c4.err; echo "c4 rc=$?"
timeout 600 python bench.py --workload c2 --steps 10 --warmup 3 > gpurun_out/r79_bench_c2.json 2> gpurun_out/r79_bench_c2.err; echo "c2 rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r79_bench_ref.json 2> gpurun_out/r79_bench_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r79_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-secondary --no-cpu-baseline > gpurun_out/r79_ncu.log 2>&1; echo "ncu rc=$?"
