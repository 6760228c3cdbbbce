#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck) over the engine's kernel
# variants: smoke() shapes, the calendar batch (G*B > 4096: every policy,
# int32 chain, noisy producer/consumer), wide trajectories (G > 128 chains)
mkdir -p gpurun_out
OUT=gpurun_out/sanitizer.txt
: > $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
run() {  # tool, label, command...
  local tool=$1 label=$2; shift 2
  local log=gpurun_out/san_${tool}_$(echo $label | cut -c1-8 | tr -c 'a-z0-9\n' '_').log
  echo "== $tool: $label" >> $OUT
  timeout 900 $CS --tool $tool --print-limit 10 "$@" > $log 2>&1
  echo "   exit $?" >> $OUT
  grep -E "SUMMARY|rror|smoke ok|traj" $log | tail -4 >> $OUT
}
for tool in memcheck racecheck synccheck; do
  run $tool "smoke (fcfs, jsq, greedy H=0/4, noisy H=8, calendar, overloaded)" python -c "import __graft_entry__ as g; g.smoke()"
  run $tool "calendar batch (8 kernel groups incl. noisy and int32 chains)" python tools/repro_cal.py
  run $tool "wide chain (4 x G=300 B=16 H=3)" python tools/repro_wide2.py 4 300
done
cat $OUT
