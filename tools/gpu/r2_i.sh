# body diagonals at 10 warps per CTA (no row prefetch, 168 registers) against the 8-warp build
set -x
timeout 900 python -m pytest tests/test_gpu_lattice.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2i_quick.log 2>&1; rc=$?; echo "quick rc=$rc"
if [ $rc -ne 0 ]; then exit 1; fi
for L in D3Q15 D3Q27; do
  timeout 600 python bench.py --lattice $L --cells 128 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2i_lat_$L.json 2>&1
done
