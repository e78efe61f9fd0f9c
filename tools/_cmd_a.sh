timeout 900 python -m pytest tests/test_ttc_gpu.py -m gpu -x -q 2>&1 | tail -3
python tools/prof_cfg5.py 128; python tools/prof_cfg5.py 128
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:ms_epi -c 2 python tools/prof_cfg5.py 128 2>&1 | grep -E "duration"
