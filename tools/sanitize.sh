#!/bin/bash
# compute-sanitizer (memcheck / racecheck / synccheck / initcheck) over smoke():
# every kernel family the bench times, at small shapes.  Summaries -> gpurun_out/san_*.txt
O=gpurun_out; mkdir -p $O
for tool in memcheck synccheck racecheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 \
    python -c "import __graft_entry__ as g; g.smoke()" > $O/san_$tool.txt 2>&1
  echo "$tool rc=$?" | tee -a $O/san_$tool.txt
  tail -3 $O/san_$tool.txt
done
