#!/bin/bash
# small-kernel column-split sweep + K2000 timing
for cs in 1 2 4; do echo "cs=$cs"; NMFA_SMALL_CS=$cs timeout 120 python tools/probe.py sk100; done
timeout 200 python tools/probe.py k2000
