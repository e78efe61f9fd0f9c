timeout 900 python -m pytest tests/test_ttc_gpu.py -m gpu -x -q 2>&1 | tail -3
python tools/time_moments.py 256 f64; python tools/time_moments.py 256 f64
