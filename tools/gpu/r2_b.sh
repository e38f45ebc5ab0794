set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
PDG_FUZZ_SEEDS_BACKWARD=400 timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rs \
    > gpurun_out/r2b_pytest.log 2>&1; echo "pytest rc=$?"
PDG_FUZZ_SEEDS_BACKWARD=400 timeout 600 python -m pytest tests/test_gpu_fuzz.py -m gpu -q -s -k backward -p no:cacheprovider \
    2>&1 | grep "^backward" > gpurun_out/r2b_backward.txt
bash tools/gpu/parity_long.sh cfg2,cfg3,cfg2s,cfg3s 2400
