export CT_CONV_TXN=8 CT_CONV_TYN=32
python tools/prof_conv.py cfg4 2 > gpurun_out/c4plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:xcorr -s 2 -c 1 -o gpurun_out/prof_c4pair2 python tools/prof_conv.py cfg4 1 > /dev/null 2>&1; echo done
