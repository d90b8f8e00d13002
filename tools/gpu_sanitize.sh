# ONE compute-sanitizer tool per gpurun call (B200_PROFILING.md: several tools in one
# call have left a GPU unusable).  usage: bash tools/gpu_sanitize.sh <tool> [c2_frames]
TOOL=$1; N=${2:-200}
mkdir -p gpurun_out/r2/sanitizer
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python tools/sanitize_run.py $N > gpurun_out/r2/sanitizer/plain_$TOOL.log 2>&1
echo "plain rc=$?"
EXTRA=""
[ "$TOOL" = racecheck ] && EXTRA="--racecheck-report all"
timeout 2400 /usr/local/cuda/bin/compute-sanitizer --tool $TOOL $EXTRA --error-exitcode 9 \
  python tools/sanitize_run.py $N > gpurun_out/r2/sanitizer/$TOOL.log 2>&1
echo "$TOOL rc=$?"; tail -5 gpurun_out/r2/sanitizer/$TOOL.log
