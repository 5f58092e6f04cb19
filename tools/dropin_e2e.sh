#!/bin/bash
# The reference's own pipeline.cpp::decompose, unchanged, linked against the
# drop-in (cp_e2e) and against the reference library itself (cp_e2e_ref).
mkdir -p gpurun_out
B=integration/_build
run() {  # name args...
  local name=$1; shift
  echo "{\"case\": \"$name\", \"args\": \"$*\", \"impl\": \"xtsg\"}" >> gpurun_out/dropin.jsonl
  timeout 600 $B/cp_e2e "$@" >> gpurun_out/dropin.jsonl 2>> gpurun_out/dropin.err
  echo "{\"case\": \"$name\", \"args\": \"$*\", \"impl\": \"reference\", \"threads\": $(nproc)}" >> gpurun_out/dropin.jsonl
  timeout 900 $B/cp_e2e_ref "$@" >> gpurun_out/dropin.jsonl 2>> gpurun_out/dropin.err
}
rm -f gpurun_out/dropin.jsonl gpurun_out/dropin.err
run C1 200 30 10 12 10 tensor 3
run dense400 400 30 10 20 10 tensor 2
run factors1000 1000 40 20 56 20 factors 1
cat gpurun_out/dropin.jsonl
