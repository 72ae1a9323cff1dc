# compute-sanitizer over every k_guiding_pass instantiation (tools/sanitize_pass.py)
set -u
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for t in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $t --error-exitcode 9 --print-limit 50 python tools/sanitize_pass.py > gpurun_out/sanitize_$t.log 2>&1
  echo $t=$?
done
