for W in 4,2 2,4 1,8; do PDG_LATTICE_WARPS=$W timeout 600 python bench.py --lattice D3Q15 --cells 128 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/shape_D3Q15_w$W.json 2>&1; done
for W in 8,1 4,2 2,4; do PDG_LATTICE_WARPS=$W timeout 600 python bench.py --lattice D3Q19 --cells 128 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/shape_D3Q19_w$W.json 2>&1; done
echo done
