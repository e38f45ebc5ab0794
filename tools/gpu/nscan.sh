timeout 900 python -m pytest tests/test_gpu_lattice.py tests/test_gpu_source.py tests/test_gpu_fuzz.py tests/test_gpu_fullsize.py -q -x -k "not cfg and not fullsize_one_step and not fused_passes" 2>&1 | tail -2
for L in D3Q15 D3Q19 D3Q27; do timeout 600 python bench.py --lattice $L --cells 128 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ns3_$L.json 2>&1; done
timeout 600 python bench.py --lattice D2Q9 --cells 1024 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ns3_D2Q9.json 2>&1
echo done
