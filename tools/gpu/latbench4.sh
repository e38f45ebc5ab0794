timeout 600 python -m pytest tests/test_gpu_lattice.py -q -x 2>&1 | tail -2
for L in D3Q15 D3Q19 D3Q27; do timeout 600 python bench.py --lattice $L --cells 128 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/lat4_$L.json 2> gpurun_out/lat4_$L.err; done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:lattice_sweep_kernel -s 6 -c 1 -o gpurun_out/lat_act7 python bench.py --lattice D3Q15 --cells 128 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_act7.log 2>&1
echo done
