cd tools/micro && bash build.sh > /dev/null 2>&1; ./pipes > ../../gpurun_out/g3_pipes.log 2>&1; cd ../..
cat gpurun_out/g3_pipes.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:small_solve_tc -c 1 -o gpurun_out/g3_c4 -f python tools/ncu_driver.py c4 2 > gpurun_out/g3_ncu_c4.log 2>&1; echo "ncu c4 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:proj_kernel -c 1 -o gpurun_out/g3_proj -f python tools/ncu_driver.py c5 1 > gpurun_out/g3_ncu_proj.log 2>&1; echo "ncu proj rc=$?"
