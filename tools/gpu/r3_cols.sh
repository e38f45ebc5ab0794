# config 2's y sweeps: persistent double-buffered tile kernel (sweep_cols) -- parity + bench + ncu
set -x
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/c3_pytest.log 2>&1; echo "pytest rc=$?"
PDG_CHECKED=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "strided or tile or cols or fused" > gpurun_out/c3_pytest_checked.log 2>&1; echo "checked rc=$?"
for k in 1 2; do timeout 600 python bench.py --config 2 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/c3_cfg2_$k.json 2>&1; done
timeout 600 python bench.py --config 3 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/c3_cfg3.json 2>&1
timeout 600 python bench.py --config 1 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/c3_cfg1.json 2>&1
CMD="python bench.py --config 2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sweep_cols|relax_xsweep" -s 8 -c 2 \
    -o gpurun_out/c3_ncu_cfg2 $CMD > gpurun_out/c3_ncu.log 2>&1; echo "ncu rc=$?"
