timeout 900 ncu --set full --clock-control none -k regex:lattice_sweep_kernel -s 0 -c 1 -o gpurun_out/lat_act3 python bench.py --lattice D3Q19 --cells 128 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_act3.log 2>&1
echo done
