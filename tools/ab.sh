#!/bin/bash
# A/B timing of the argmax step on one box: alternates the default libsecpe.so and a variant
# (paper_2502_00847_b200/libsecpe_<variant>.so), R rounds each.
#   usage: tools/ab.sh <variant> [rounds] [batch] [streams]
V=$1; R=${2:-3}; B=${3:-16}; S=${4:-2}
for i in $(seq 1 $R); do
  for lib in libsecpe.so libsecpe_$V.so; do
    ms=$(SECPE_STREAMS=$S SECPE_LIB=paper_2502_00847_b200/$lib SECPE_BATCH=$B timeout 300 python tools/microbench.py argmax --reps 6 2>/dev/null | grep ms_per_batch | tr -dc '0-9.')
    echo "$lib S=$S $ms"
  done
done
