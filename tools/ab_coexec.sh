#!/bin/bash
# concurrent parts with a persistent vs a wave-scheduled K4
for t in 0 16 4; do echo "K4_TPW=$t"; PJG_K4_TPW=$t timeout 600 python tools/streams_probe.py 2>&1 | tail -5; done
