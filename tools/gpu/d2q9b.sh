timeout 600 python -m pytest tests/test_gpu_lattice.py tests/test_gpu_source.py -q -x 2>&1 | tail -2
timeout 600 python bench.py --lattice D2Q9 --cells 1024 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/d2q9b.json 2>&1
timeout 600 python bench.py --lattice D2Q9 --cells 2048 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/d2q9b_2048.json 2>&1
timeout 600 python bench.py --lattice D3Q19 --cells 128 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/d3q19b.json 2>&1
echo done
