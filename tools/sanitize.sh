#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck on smoke() and on one
# fwd+bwd per kernel path; logs to gpurun_out/sanitizer_*.txt (summaries go to profiles/).
# TOOLS overrides the tool list (default: memcheck racecheck synccheck).
set -u
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
run() {  # name tool cmd...
  local name=$1 tool=$2; shift 2
  timeout ${ST:-1200} $CS --tool $tool --print-limit 20 "$@" > gpurun_out/sanitizer_${name}_${tool}.txt 2>&1
  echo "== $name $tool rc=$? :: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard|Error' gpurun_out/sanitizer_${name}_${tool}.txt | tail -2 | tr '\n' ' ')"
}
for tool in ${TOOLS:-memcheck racecheck synccheck}; do
  run smoke $tool python -c "import __graft_entry__ as g; g.smoke()"
  # staged dE (S <= 832), multi-pass dH (V = 100000 at D = 768: 4 passes), 2-CTA forward, MXFP8 forward
  run staged $tool python tools/sanitize_case.py 4 512 768 100000 0 mx
  # sparse regime (bias -2: a few % active pairs): sparse dE, single-pass dH; MXFP8 packed short sequences
  run sparse $tool python tools/sanitize_case.py 4 512 768 100000 -2
  # gathered dE (S > 832) and packed short sequences
  run gathered $tool python tools/sanitize_case.py 3 1000 256 20000
  run packed $tool python tools/sanitize_case.py 16 48 128 5000 0 mx
  # the peer-memory dH reduction kernel
  run allreduce $tool python tools/sanitize_allreduce.py
done
