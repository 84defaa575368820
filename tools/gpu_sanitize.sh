# compute-sanitizer over smoke() (one tcgen05 GEMM + one tiny bf16 Adam BERT step
# through the device VM, ~43 kernels): memcheck, racecheck, synccheck.
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
    python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_summary.txt
  tail -n 4 gpurun_out/sanitize_$tool.log >> gpurun_out/sanitize_summary.txt
done
cat gpurun_out/sanitize_summary.txt
