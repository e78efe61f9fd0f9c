# Profiling pass for profiles/ (one ncu per gpurun call): plain bench run,
# which must exit 0, then the ncu launch list of the same command.  The full
# per-kernel captures come from a separate call:
#   ncu --set full --clock-control none --import-source on \
#       -k regex:"ttc_moments_kernel|xcorr_zwalk|xcorr_pair|blur5" -c 5 -o gpurun_out/prof_all python tools/prof_all.py
set -e
python bench.py --steps 2 --warmup 3 --cpu-seconds 1 --no-secondary > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/bench_launches.csv \
    python bench.py --steps 2 --warmup 3 --cpu-seconds 1 --no-secondary > gpurun_out/ncu_list.log 2>&1
echo done
