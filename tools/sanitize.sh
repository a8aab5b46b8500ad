#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over every kernel family
# at small shapes (tools/sanitize_run.py).  Run on the GPU box from the repo
# root; writes one log per (tool, part) plus summary.txt to gpurun_out/sanitize/.
OUT=gpurun_out/sanitize
mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
PARTS="score_fused score_multi score_fused256 score_multi256 select compress_decode decode_coop decode_wide decode_solo exchange"
: > $OUT/summary.txt
for tool in memcheck racecheck synccheck initcheck; do
  for part in $PARTS; do
    extra=""
    [ $tool = memcheck ] && extra="--leak-check no"
    [ $tool = racecheck ] && extra="--racecheck-report all"
    timeout 900 $CS --tool $tool $extra --error-exitcode 9 python tools/sanitize_run.py $part \
      > $OUT/${tool}_${part}.log 2>&1
    rc=$?
    res=$(grep -E "ERROR SUMMARY|RACECHECK SUMMARY|hazard|Error" $OUT/${tool}_${part}.log | tail -2 | tr '\n' ' ')
    ok=$(grep -E "^\[$part\]" $OUT/${tool}_${part}.log | tail -1)
    echo "$tool $part rc=$rc | $res | $ok" >> $OUT/summary.txt
  done
done
cat $OUT/summary.txt
