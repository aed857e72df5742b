#!/bin/bash
# A/B timing of alternative builds (tools/libgsr_*.so) against the in-tree library
python tools/quick_time.py C4 C5s
for f in tools/libgsr_E*.so; do echo "== $f"; GSR_LIB_PATH=$f python tools/quick_time.py C4 C5s; done
echo "== base again"; python tools/quick_time.py C4 C5s
