# CTA shape sweep of the segmented 2-D diagonal sweep
for W in 8,1 4,1 2,1 1,1; do for N in 1024 2048; do
timeout 300 python bench.py --lattice-cta $W --lattice D2Q9 --cells $N --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ws_${W}_$N.json 2> gpurun_out/ws_${W}_$N.err
done; done
echo done
