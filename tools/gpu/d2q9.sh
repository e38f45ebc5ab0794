for W in 8,1 4,1 2,1; do PDG_LATTICE_WARPS=$W timeout 600 python bench.py --lattice D2Q9 --cells 1024 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/d2q9_w$W.json 2>&1; done
for W in 8,1 4,1; do PDG_LATTICE_WARPS=$W timeout 600 python bench.py --lattice D2Q9 --cells 2048 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/d2q9_2048_w$W.json 2>&1; done
echo done
