CT_NO_BM=1 python tools/bm_check.py save && python tools/bm_check.py compare
timeout 900 python -m pytest tests/test_ttc_gpu.py -m gpu -x -q 2>&1 | tail -3
python tools/prof_cfg5.py 128; python tools/prof_cfg5.py 128
ncu --metrics gpu__time_duration.sum --clock-control none -c 12 --csv --log-file gpurun_out/launches5.csv python tools/prof_cfg5.py 128 > /dev/null 2>&1
