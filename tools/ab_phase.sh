#!/bin/bash
# A/B of alternative builds (tools/libgsr_E*.so) against the in-tree library, per phase
CFGS=${CFGS:-"C2 C4 C5s"}
python tools/phase_time.py $CFGS
for f in tools/libgsr_E*.so; do echo "== $f"; GSR_LIB_PATH=$f python tools/phase_time.py $CFGS; done
echo "== base again"; python tools/phase_time.py $CFGS
