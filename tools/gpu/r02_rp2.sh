# checkpointed projection sweeps: GPU suite after the outside-m delta fix
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/rp2_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/rp2_tests.log
python -m pytest tests/test_gpu_fullsize_lockstep.py -q -s -k "lockstep and not sums" 2>&1 | grep -E "max|passed|failed" | tail -8
