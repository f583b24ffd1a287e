timeout 900 ncu --set full --import-source on --clock-control none -k regex:proj_kernel -s 1 -c 1 -o gpurun_out/r72_proj python tools/prec_time.py c5 3 > gpurun_out/r72_ncu.log 2>&1; echo "ncu rc=$?"
