for cfg in "CT_MOM_RS=1" "CT_MOM_RS=2" "CT_MOM_SYNC=1"; do
  echo "== $cfg"
  env $cfg python tools/time_moments.py 256 f32
  env $cfg python tools/time_moments.py 2 f32 1080 1920 128
done
CT_MOM_RS=2 timeout 600 python -m pytest tests/test_ttc_gpu.py -m gpu -x -q 2>&1 | tail -3
CT_MOM_RS=1 timeout 600 python -m pytest tests/test_ttc_gpu.py -m gpu -x -q 2>&1 | tail -3
