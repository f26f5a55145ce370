#!/usr/bin/env bash
# Round measurement on one B200 (run through gpurun from the repo root):
#   1. bench.py as the driver runs it (no profiler)      -> gpurun_out/bench_<tag>.json
#   2. the launch list of the same command under ncu      -> gpurun_out/launches_<tag>.csv
#   3. one `--set full` capture of the first rasteriser   -> gpurun_out/raster_full_<tag>.ncu-rep
# Steps 2-3 run only after step 1 exited 0. Summaries: scripts/summarize_ncu.py.
# (The first rasteriser launch of a fresh context is an aborted capacity probe that
# the step replays with exact sizes: the full capture skips it.)
set -euo pipefail
TAG=${1:-r}
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
tail -1 gpurun_out/bench_${TAG}.json
ARGS="--steps 2 --warmup 1 --no-e2e --no-optim --no-io --no-c4 --no-det --no-c2 --no-c5 --cpu-seconds 0 --sweep= --precision-sweep= --no-refbench"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_${TAG}.csv python bench.py $ARGS > gpurun_out/ncu_launch_${TAG}.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_raster_resident -s 1 -c 1 \
    -o gpurun_out/raster_full_${TAG} -f python bench.py $ARGS > gpurun_out/ncu_full_${TAG}.log 2>&1
echo "profiles done"
