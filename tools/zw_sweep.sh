#!/bin/bash
# z-walk conv configurations on cfg3 (+ cfg4 pair kernel check)
for c in 0 1 2; do echo -n "kind 4 cfg $c: "; CT_CONV_KIND=4 CT_ZW_CFG=$c python tools/prof_conv.py cfg3 5; done
for c in 0 2; do echo -n "kind 5 cfg $c: "; CT_CONV_KIND=5 CT_ZW_CFG=$c python tools/prof_conv.py cfg3 5; done
echo -n "auto: "; python tools/prof_conv.py cfg3 5
echo -n "cfg4 auto: "; python tools/prof_conv.py cfg4 5
