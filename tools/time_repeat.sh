#!/bin/bash
# run quick_time several times to see run-to-run variance
for i in 1 2 3; do python tools/quick_time.py C5s; done
