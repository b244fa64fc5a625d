#!/bin/bash
for sp in "1 4" "2 4" "3 8"; do set -- $sp; SP1=$1 SP2=$2 timeout 120 python tools/k2_run.py; done
