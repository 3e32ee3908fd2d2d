# round 2, call AC: compute-sanitizer (memcheck / racecheck / synccheck) over every kernel incl. the TMA Radon
# kernel and the fused P stage; TMA Radon timings of the current build
mkdir -p gpurun_out/r02ac
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/r02ac
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_cases.py > $O/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 $O/sanitize_$tool.log
done
