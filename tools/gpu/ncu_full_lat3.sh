# ncu --set full of the final body-diagonal sweep and the two-phase LBM relaxation (D3Q15 128^3)
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"lattice_sweep_kernel<\(int\)3, \(int\)3, \(int\)7" -s 2 -c 1 -o gpurun_out/lat_act7_v3 python bench.py --lattice D3Q15 --cells 128 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_act7_v3.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"relax_lbm2_kernel" -s 2 -c 1 -o gpurun_out/lat_relax2_v1 python bench.py --lattice D3Q15 --cells 128 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_relax2.log 2>&1
echo done
