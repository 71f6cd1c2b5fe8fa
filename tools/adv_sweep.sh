#!/bin/bash
# advance-kernel lane-group sweep on C2 (timing probe per AKNN_ADV_BPL value)
for b in 4 8 16 32 64 128; do
  echo "bpl=$b $(AKNN_ADV_BPL=$b python tools/timing_probe.py 2>&1 | grep host_t1)"
done
