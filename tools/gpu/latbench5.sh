timeout 600 python -m pytest tests/test_gpu_lattice.py tests/test_gpu_source.py -q -x 2>&1 | tail -2
for L in D3Q15 D3Q19 D3Q27; do timeout 600 python bench.py --lattice $L --cells 128 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/lat5_$L.json 2> gpurun_out/lat5_$L.err; done
for W in 4,1 2,2 2,1 1,2; do PDG_LATTICE_WARPS=$W timeout 600 python bench.py --lattice D3Q15 --cells 128 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/lat5_D3Q15_w$W.json 2>&1; done
for W in 4,2 2,4 1,4; do PDG_LATTICE_WARPS=$W timeout 600 python bench.py --lattice D3Q19 --cells 128 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/lat5_D3Q19_w$W.json 2>&1; done
echo done
