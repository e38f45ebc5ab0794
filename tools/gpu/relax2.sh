# two-phase LBM relaxation (PDG_LBM_RELAX2=1) against the one-read kernel
for R in 0 1; do for L in D3Q15 D3Q19 D3Q27; do
PDG_LBM_RELAX2=$R timeout 300 python bench.py --lattice $L --cells 128 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2_${R}_$L.json 2>/dev/null
done; done
echo done
