timeout 900 python -m pytest tests/test_gpu_lattice.py tests/test_gpu_source.py -q -x 2>&1 | tail -3
timeout 600 python bench.py --lattice D3Q15 --cells 64 --degree 3 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/p3_D3Q15.json 2>&1
echo done
