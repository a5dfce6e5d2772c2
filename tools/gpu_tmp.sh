set -x
python tools/poison_probe.py 2>&1 | tail -12
timeout 600 python -m pytest tests/test_gpu_traffic.py tests/test_gpu_parity.py -q -k "poison or traffic" 2>&1 | tail -4
