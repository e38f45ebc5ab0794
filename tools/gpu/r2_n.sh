# strided sweep with pointer-walk addressing
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_kernels.py tests/test_gpu_fullsize.py tests/test_gpu_lattice.py -m gpu -q -x -p no:cacheprovider \
    > gpurun_out/r2n_quick.log 2>&1; rc=$?; echo "quick rc=$rc"
if [ $rc -ne 0 ]; then exit 1; fi
for c in 3 4; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2n_cfg$c.json 2>&1
done
for k in 1 2; do timeout 900 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2n_bench_$k.json 2>&1; done
