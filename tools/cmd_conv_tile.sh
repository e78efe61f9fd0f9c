for c in cfg4 cfg3; do
python tools/prof_conv.py $c 5
for t in "16 16" "32 8" "16 8" "8 32" "32 4"; do set -- $t; echo -n "txn=$1 tyn=$2 "; CT_CONV_TXN=$1 CT_CONV_TYN=$2 python tools/prof_conv.py $c 5; done
done
