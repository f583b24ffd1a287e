# The round-end GPU run (gpurun -- bash tools/gpu/round_end.sh): GPU tests, smoke, the bench lines
# (c5 default, c4, c2 on c5's fixed schedule, the oracle reference arm), the ncu launch list of the
# bench command (only after the same command exited 0 without ncu) and one `ncu --set full` capture
# per top kernel. Outputs land in gpurun_out/ (TAG prefix).
T=${TAG:-round_end}
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/${T}_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --workload c4 --steps 400 --warmup 3 > gpurun_out/${T}_bench_c4.json 2> gpurun_out/${T}_bench_c4.err; echo "c4 rc=$?"
timeout 600 python bench.py --workload c2 --steps 10 --warmup 3 > gpurun_out/${T}_bench_c2.json 2> gpurun_out/${T}_bench_c2.err; echo "c2 rc=$?"
timeout 1200 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${T}_bench_ref.json 2> gpurun_out/${T}_bench_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-secondary --no-cpu-baseline > gpurun_out/${T}_ncu.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_i8_kernel -c 1 -o gpurun_out/${T}_gemm_i8 -f python tools/ncu_driver.py c5 1 > gpurun_out/${T}_ncu_gemm.log 2>&1; echo "ncu gemm rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:proj_kernel -c 1 -o gpurun_out/${T}_proj -f python tools/ncu_driver.py c5 1 > gpurun_out/${T}_ncu_proj.log 2>&1; echo "ncu proj rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:small_solve_tc -c 1 -o gpurun_out/${T}_c4 -f python tools/ncu_driver.py c4 20 > gpurun_out/${T}_ncu_c4.log 2>&1; echo "ncu c4 rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:rounds_kernel -c 1 -o gpurun_out/${T}_greedy -f python tools/ncu_driver.py discretize 16384 > gpurun_out/${T}_ncu_greedy.log 2>&1; echo "ncu greedy rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:proj_onchip_kernel -c 1 -o gpurun_out/${T}_onchip -f python tools/ncu_driver.py c2 1 > gpurun_out/${T}_ncu_onchip.log 2>&1; echo "ncu onchip rc=$?"
