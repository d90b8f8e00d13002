# Memory / hand-off checking of every kernel of the path.  compute-sanitizer is closed on
# this pool, so this runs tools/sanitize_run.py on the bounds-checked build of the library
# (-DCLIPDETECT_CHECKED, common.cuh CD_CHECK) after the same run on the product build.
# usage: bash tools/gpu_sanitize.sh [c2_frames]    (logs in gpurun_out/r2/sanitizer/)
N=${1:-200}
mkdir -p gpurun_out/r2/sanitizer
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python tools/sanitize_run.py $N > gpurun_out/r2/sanitizer/product.log 2>&1
echo "product rc=$?"; tail -2 gpurun_out/r2/sanitizer/product.log
timeout 1800 python tools/sanitize_run.py $N --checked > gpurun_out/r2/sanitizer/checked.log 2>&1
echo "checked rc=$?"; tail -3 gpurun_out/r2/sanitizer/checked.log
