#!/bin/bash
# A/B timing of alternative builds (tools/libgsr_E*.so) against the in-tree library
CFGS=${CFGS:-"C4 C5s"}
python tools/quick_time.py $CFGS
for f in tools/libgsr_E*.so; do echo "== $f"; GSR_LIB_PATH=$f python tools/quick_time.py $CFGS; done
echo "== base again"; python tools/quick_time.py $CFGS
