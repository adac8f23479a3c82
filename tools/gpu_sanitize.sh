# compute-sanitizer over every kernel (tools/sanitize.py); logs -> gpurun_out/sanitizer_<tool>.txt
python tools/sanitize.py > gpurun_out/sanitize_plain.txt 2>&1; echo "plain rc=$?" >> gpurun_out/sanitize_plain.txt
for t in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 50 --target-processes all python tools/sanitize.py > gpurun_out/sanitizer_$t.txt 2>&1
  echo "tool=$t rc=$?" >> gpurun_out/sanitizer_$t.txt
done
tail -n 4 gpurun_out/sanitize_plain.txt gpurun_out/sanitizer_*.txt
