# segment length sweep of the 2-D diagonal sweep
for L in 32 48 64 96; do timeout 300 python bench.py --lattice-segment $L --lattice D2Q9 --cells 1024 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ss_${L}_1024.json 2>/dev/null; done
for L in 64 96 128 160; do timeout 300 python bench.py --lattice-segment $L --lattice D2Q9 --cells 2048 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ss_${L}_2048.json 2>/dev/null; done
echo done
