timeout 900 python -m pytest tests/test_gpu_lattice.py tests/test_gpu_source.py tests/test_gpu_fuzz.py -q -x 2>&1 | tail -2
for L in D3Q19 D3Q27 D3Q15; do timeout 600 python bench.py --lattice $L --cells 128 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/gs_$L.json 2>&1; done
timeout 600 python bench.py --lattice D2Q9 --cells 1024 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/gs_D2Q9.json 2>&1
echo done
