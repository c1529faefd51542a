#!/bin/bash
# A/B device timing of library variants on config 5: tools/ab.sh lib1.so lib2.so ... (alternating, 2 rounds)
for r in 1 2; do for L in "$@"; do echo "== $L"; HMMSCAN_LIB=$L python tools/t8.py; done; done
