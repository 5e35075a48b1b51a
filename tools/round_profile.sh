#!/usr/bin/env bash
# One GPU call that refreshes every judged artefact (run under gpurun):
#   gpu tests, bench (both arms), ncu launch list of the bench command, one
#   ncu --set full capture of the headline expand launch.
# Usage: gpurun --timeout 2400 -- 'bash tools/round_profile.sh TAG'
set -u
TAG=${1:-r01}
O=gpurun_out/$TAG
mkdir -p "$O"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > "$O/gpu.txt" 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > "$O/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$O/pytest_gpu.log"
timeout 600 python bench.py > "$O/bench.json" 2> "$O/bench.err"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > "$O/bench_reference.json" 2> "$O/bench_reference.err"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file "$O/launches.csv" python bench.py --steps 2 --warmup 3 --no-cpu-baseline > "$O/launches_bench.log" 2>&1
# headline kernel: expand_tma_kernel<2> of the idx (decompress_chunked) plans.  The
# no-index plans are timed first (one launch per step: 3 warmup + 1 timed), so skip 5.
timeout 900 ncu --set full --clock-control none --import-source on -k regex:expand_tma_kernel -s 5 -c 1 \
    -o "$O/full_expand" -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-extras \
    > "$O/full_expand.log" 2>&1

# fused decompress -> GEMV (one batched launch per layer) and the batched dense GEMV
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv_fused_kernel -c 1 \
    -o "$O/full_fused" -f python tools/fused_bench.py > "$O/full_fused.log" 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv_batch_kernel -c 1 \
    -o "$O/full_gemv" -f python tools/fused_bench.py > "$O/full_gemv.log" 2>&1
timeout 300 python tools/fused_bench.py > "$O/fused_bench.log" 2>&1
timeout 300 python tools/extract_probe.py > "$O/extract.log" 2>&1 && cp gpurun_out/extract_probe.json "$O/extract.json"
echo done2
# r02 additions: secondary paths (clean L2 flush), small shards, coarse-index and count timings,
# and an ncu capture of the coarse-index (chunk 4096) expand
timeout 300 python tools/secondary_kernels.py --out "$O/secondary.json" > "$O/secondary.log" 2>&1
timeout 600 python tools/small_shards.py --reps 20 --out "$O/small_shards.json" > "$O/small_shards.log" 2>&1
timeout 300 python tools/chunked_time.py > "$O/chunked_time.txt" 2>&1
timeout 300 python tools/count_time.py > "$O/count_time.txt" 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:expand_tma_kernel -s 2 -c 1 \
    -o "$O/full_expand_chunk4096" -f python tools/chunked_one.py 4096 > "$O/full_expand_chunk4096.log" 2>&1
echo done3
