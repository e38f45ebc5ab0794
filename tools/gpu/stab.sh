for rep in 1 2; do timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -1; done
for L in D3Q15 D3Q19 D3Q27; do timeout 600 python bench.py --lattice $L --cells 128 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ypf3_$L.json 2>&1; done
for L in D3Q19 D3Q27; do PDG_LATTICE_NOYPF=1 timeout 600 python bench.py --lattice $L --cells 128 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/noypf3_$L.json 2>&1; done
echo done
