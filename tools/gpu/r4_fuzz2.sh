# 4000/1000/1000-seed fuzz campaigns with the conditioning-aware bars (reading C29), then the
# source-level ncu capture of the body-diagonal sweep
set -x
PDG_FUZZ_SEEDS_MAIN=4000 PDG_FUZZ_SEEDS_BACKWARD=1000 PDG_FUZZ_SEEDS=1000 timeout 3000 python -m pytest tests/test_gpu_fuzz.py -m gpu -q -s \
    -p no:cacheprovider -rs > gpurun_out/f5_fuzz.log 2>&1; echo "fuzz rc=$?"
grep -E 'forward|backward' gpurun_out/f5_fuzz.log | head -40
tail -n 3 gpurun_out/f5_fuzz.log
bash tools/gpu/r4_latsrc.sh
