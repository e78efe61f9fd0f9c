# Profiling pass for profiles/: plain bench run (must exit 0), then the ncu
# launch list of the same command, then one full capture of the top kernel.
set -e
python bench.py --steps 2 --warmup 3 --cpu-seconds 1 --no-secondary > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/bench_launches.csv \
    python bench.py --steps 2 --warmup 3 --cpu-seconds 1 --no-secondary > gpurun_out/ncu_list.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:ttc_moments -s 0 -c 1 -o gpurun_out/bench_moments \
    python bench.py --steps 2 --warmup 3 --cpu-seconds 1 --no-secondary > gpurun_out/ncu_full.log 2>&1
echo done
