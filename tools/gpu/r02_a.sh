set -x
timeout 600 python -m pytest tests/test_gpu_api.py tests/test_gpu_fullsize_lockstep.py::test_c5_full_size_sweep_sums -x -q -s > gpurun_out/g1_api.log 2>&1; echo "api rc=$?"; tail -5 gpurun_out/g1_api.log
timeout 1500 python -m pytest tests -m gpu -q --deselect tests/test_gpu_fullsize_lockstep.py::test_c5_full_size_lockstep > gpurun_out/g1_suite.log 2>&1; echo "suite rc=$?"; tail -15 gpurun_out/g1_suite.log
FASTPFP_FULLSIZE_ITERS=10 FASTPFP_FULLSIZE_GREEDY=1 FASTPFP_LOCKSTEP_OUT=gpurun_out/r02_c5_lockstep.json timeout 2400 python -m pytest tests/test_gpu_fullsize_lockstep.py::test_c5_full_size_lockstep -x -q -s > gpurun_out/g1_lock.log 2>&1; echo "lock rc=$?"; tail -20 gpurun_out/g1_lock.log
