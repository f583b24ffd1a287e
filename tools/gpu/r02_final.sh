# final round-2 set: the standard round-end script, then the 10-iteration full-size lockstep record
TAG=r02f bash tools/gpu/round_end.sh
FASTPFP_FULLSIZE_ITERS=10 FASTPFP_FULLSIZE_GREEDY=1 FASTPFP_LOCKSTEP_OUT=gpurun_out/r02f_c5_lockstep.json timeout 2400 python -m pytest tests/test_gpu_fullsize_lockstep.py::test_c5_full_size_lockstep -x -q -s > gpurun_out/r02f_lock.log 2>&1; echo "lock rc=$?"; tail -3 gpurun_out/r02f_lock.log
