# ncu --set full of the current body-diagonal sweep (D3Q15 128^3) and the segmented 2-D diagonal sweep (D2Q9 1024^2)
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"lattice_sweep_kernel<\(int\)3, \(int\)3, \(int\)7" -s 2 -c 1 -o gpurun_out/lat_act7_v2 python bench.py --lattice D3Q15 --cells 128 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_act7_v2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"lattice_sweep_kernel<\(int\)2, \(int\)3, \(int\)3" -s 2 -c 1 -o gpurun_out/lat_2d_v2 python bench.py --lattice D2Q9 --cells 1024 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_2d_v2.log 2>&1
echo done
