# Round profile capture (run on the GPU box from the repo root):
#   bash scripts/capture_profiles.sh <tag>
# Writes ncu reports and launch lists under gpurun_out/; scripts/summarize_profiles.py
# turns them into the tracked summaries under profiles/.
tag=${1:-r01}
set -x
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/${tag}_bench_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:kv_tc_kernel -s 2 -c 1 \
  -o gpurun_out/${tag}_kv_c2_m32 python scripts/kv_profile.py --config 2 --m 32 --reps 1 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:kv_tc_kernel -s 2 -c 1 \
  -o gpurun_out/${tag}_kv_c2_m266 python scripts/kv_profile.py --config 2 --m 266 --reps 1 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:kv_tc_kernel -s 1 -c 1 \
  -o gpurun_out/${tag}_kv_c3_m64 python scripts/kv_profile.py --config 3 --m 64 --reps 1 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:kv_tc_kernel -s 1 -c 1 \
  -o gpurun_out/${tag}_otf_c5_n262144 python scripts/otf_profile.py --config 5 --n 262144 --reps 1 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:kv_tc_kernel -s 1 -c 1 \
  -o gpurun_out/${tag}_otf_c4_n262144 python scripts/otf_profile.py --config 4 --n 262144 --reps 1 > /dev/null 2>&1
ls -la gpurun_out/
