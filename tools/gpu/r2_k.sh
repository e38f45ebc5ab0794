set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "standin or sharded or nccl" > gpurun_out/r2k_quick.log 2>&1; echo "rc=$?"
