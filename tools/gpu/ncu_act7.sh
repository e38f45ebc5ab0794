timeout 900 ncu --set full --import-source on --clock-control none -k regex:lattice_sweep_kernel -s 6 -c 1 -o gpurun_out/lat_act7_mma python bench.py --lattice D3Q15 --cells 128 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_act7_mma.log 2>&1
echo done
