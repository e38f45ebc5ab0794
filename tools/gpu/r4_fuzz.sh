# round-2 closing evidence: large fuzz campaigns against the oracle, the full GPU suite (default and checked builds), smoke
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f4_smoke.log 2>&1; echo "smoke rc=$?"
PDG_FUZZ_SEEDS_MAIN=4000 PDG_FUZZ_SEEDS_BACKWARD=1000 PDG_FUZZ_SEEDS=1000 timeout 3000 python -m pytest tests/test_gpu_fuzz.py -m gpu -q \
    -p no:cacheprovider -rs > gpurun_out/f4_fuzz.log 2>&1; echo "fuzz rc=$?"
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rs > gpurun_out/f4_pytest.log 2>&1; echo "pytest rc=$?"
PDG_CHECKED=1 timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rs > gpurun_out/f4_pytest_checked.log 2>&1; echo "checked rc=$?"
tail -2 gpurun_out/f4_fuzz.log gpurun_out/f4_pytest.log gpurun_out/f4_pytest_checked.log gpurun_out/f4_smoke.log
