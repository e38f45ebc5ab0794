timeout 600 python -m pytest tests/test_gpu_lattice.py tests/test_gpu_source.py -q -x 2>&1 | tail -2
for L in D3Q15 D3Q19 D3Q27; do timeout 600 python bench.py --lattice $L --cells 128 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/lat6_$L.json 2> gpurun_out/lat6_$L.err; done
PDG_LATTICE_WARPS=4,2 timeout 600 python bench.py --lattice D3Q15 --cells 128 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/lat6_D3Q15_w4,2.json 2>&1
timeout 600 python bench.py --lattice D2Q9 --cells 1024 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/lat6_D2Q9.json 2>&1
echo done
