timeout 600 python -m pytest tests/test_gpu_lattice.py tests/test_gpu_source.py -q -x 2>&1 | tail -2
for L in D3Q27 D3Q19 D3Q15; do timeout 600 python bench.py --lattice $L --cells 128 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/final2_$L.json 2>&1; done
echo done
