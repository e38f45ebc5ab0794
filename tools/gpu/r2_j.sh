# shared-memory carveout removed again (it cost relax_xsweep 0.96 -> 0.75 of HBM); 2-node batches in the
# 2-D fused pass
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_kernels.py -m gpu -q -x -p no:cacheprovider \
    > gpurun_out/r2j_quick.log 2>&1; rc=$?; echo "quick rc=$rc"
if [ $rc -ne 0 ]; then exit 1; fi
for c in 2 4; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2j_cfg$c.json 2>&1
done
timeout 900 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2j_bench.json 2>&1
