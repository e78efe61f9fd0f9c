for c in cfg1 cfg3 cfg4; do python tools/prof_conv.py $c 5; done > gpurun_out/conv_plain.log 2>&1 && cat gpurun_out/conv_plain.log && \
for c in cfg1 cfg3 cfg4; do ncu --set full --clock-control none --import-source on -k regex:xcorr -s 2 -c 1 -o gpurun_out/prof_$c python tools/prof_conv.py $c 1 > /dev/null 2>&1; done; echo done
