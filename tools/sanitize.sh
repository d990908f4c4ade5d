# compute-sanitizer passes (memcheck, racecheck, synccheck, initcheck) over smoke(): a C1 tracker
# run (graph with the conditional ICP node) plus plain fuse / raycast / ICP launches.
# usage: bash tools/sanitize.sh  -> gpurun_out/sanitize_<tool>.log
for t in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 50 --target-processes all \
    python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitize_$t.log 2>&1
  echo "$t rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|smoke ok' gpurun_out/sanitize_$t.log | tr '\n' ' ')"
done
