# round 2, first box call: build, full GPU suite (with 400 backward fuzz seeds), default bench,
# config-2 bench, z-slab emulated bench (byte accounting check)
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2a_smoke.log 2>&1; echo "smoke rc=$?"
PDG_FUZZ_SEEDS_BACKWARD=400 timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider -rs \
    > gpurun_out/r2a_pytest.log 2>&1; echo "pytest rc=$?"
timeout 600 python -m pytest tests/test_gpu_fuzz.py -m gpu -q -s -k backward -p no:cacheprovider \
    2>&1 | grep "^backward" > gpurun_out/r2a_backward.txt
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --config 2 --steps 100 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2a_cfg2.json 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --decomp zslab --slabs-per-rank 8 --no-e2e --no-cpu-baseline \
    > gpurun_out/r2a_zslab8.json 2>&1
