set -x
timeout 900 python -m pytest tests/test_grad_gpu.py -q -x 2>&1 | tail -25
