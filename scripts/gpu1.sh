set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout -s KILL 300 python -m pytest tests/test_gpu_codec.py tests/test_gpu_store.py -q -x -m gpu 2>&1 | tail -30
timeout -s KILL 200 python -m pytest tests/test_gpu_lookup.py -q -x -m gpu -k "exact_scan or golden_top1 and 1 or insert_remove or empty or topk_merge" 2>&1 | tail -30
timeout -s KILL 120 python -m pytest tests/test_gpu_lookup.py -q -x -m gpu -k "tensor_core_path_is_exact" 2>&1 | tail -30
