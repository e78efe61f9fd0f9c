python tools/prof_cfg5.py > /dev/null 2>&1 && ncu --set full --clock-control none -k regex:pyramid -s 0 -c 1 -o gpurun_out/prof_blur python tools/prof_cfg5.py > /dev/null 2>&1; echo done
