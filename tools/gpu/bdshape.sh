# CTA shape sweep of the body-diagonal (tensor-path) sweep, D3Q15 128^3
for W in 4,2 2,4 1,8 4,1 2,2; do
timeout 300 python bench.py --lattice-cta $W --lattice D3Q15 --cells 128 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bd_$W.json 2>/dev/null
done
echo done
