# tiled strided sweep with cp.async loads (8-line tiles), the TMA staging rule; quick parity + benches
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_kernels.py tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider \
    > gpurun_out/r2f_quick.log 2>&1; rc=$?; echo "quick rc=$rc"
if [ $rc -ne 0 ]; then exit 1; fi
for c in 2 3 4; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2f_cfg$c.json 2>&1
done
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --steps 10 --warmup 3 --decomp zslab --slabs-per-rank 8 --no-e2e --no-cpu-baseline \
    > gpurun_out/r2f_zslab8.json 2>&1; echo "zslab rc=$?"
timeout 300 python bench.py --config 2 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2f_cfg2b.json 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"relax_xsweep|sweep_cols" -s 6 -c 2 \
    -o gpurun_out/r2f_ncu_cfg2 python bench.py --config 2 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2f_ncu_cfg2.log 2>&1
echo "ncu rc=$?"
for L in D3Q15 D3Q19 D3Q27; do
  timeout 600 python bench.py --lattice $L --cells 128 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2f_lat_$L.json 2>&1
done
timeout 600 python bench.py --lattice D2Q9 --cells 1024 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2f_lat_D2Q9.json 2>&1
