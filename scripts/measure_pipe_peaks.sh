set -x
cd "$(dirname "$0")/.." && mkdir -p gpurun_out
(cd scripts && nvcc -O3 -gencode arch=compute_100a,code=sm_100a -I../paper_2405_03474_b200/csrc pipe_peaks.cu -o pipe_peaks)
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_throttle_reasons.active --format=csv,noheader -lms 200 > gpurun_out/peaks_clocks.csv &
SMI=$!
cd scripts && timeout 120 ./pipe_peaks > ../gpurun_out/pipe_peaks.json 2> ../gpurun_out/pipe_peaks.err
rc=$?
kill $SMI
cd ..; cat gpurun_out/pipe_peaks.json gpurun_out/pipe_peaks.err; sort gpurun_out/peaks_clocks.csv | uniq -c | sort -rn | head -8
exit $rc
