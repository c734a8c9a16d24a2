#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck) over the GPU parity suite
# (SURVEY.md 5).  The C4 case (25 M symbols, serial v1 stream) is skipped
# under the sanitizers: it only scales the same kernels up.  Logs land in
# gpurun_out/sanitize_<tool>.log; copy them to profiles/<tag>/.
mkdir -p gpurun_out
SEL=${SEL:-"not llama and not c4"}
for tool in ${TOOLS:-memcheck racecheck synccheck}; do
  extra=""
  [ "$tool" = memcheck ] && extra="--leak-check no"
  timeout ${TLIM:-1500} compute-sanitizer --tool $tool $extra --error-exitcode 17 \
      --target-processes all \
      python -m pytest tests -m gpu -x -q -k "$SEL" -p no:cacheprovider \
      > gpurun_out/sanitize_${tool}.log 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/sanitize_rc.txt
  tail -5 gpurun_out/sanitize_${tool}.log
done
