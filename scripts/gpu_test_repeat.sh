# run the GPU test suite several times (flakiness check); failures summarised
for i in 1 2 3 4 5 6 7 8; do
  timeout 400 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 > gpurun_out/rep_$i.txt; tail -1 gpurun_out/rep_$i.txt
  grep -E "^FAILED|Error|assert " gpurun_out/rep_$i.txt | head -5
done
