# which 3-D two-axis classes gain from two sweeps per launch (PDG_LATTICE_FUSE bit mask over axis masks)
for M in 104 0 64 40; do for L in D3Q19 D3Q27; do
PDG_LATTICE_FUSE=$M timeout 300 python bench.py --lattice $L --cells 128 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/fuse_${M}_$L.json 2>/dev/null
done; done
echo done
