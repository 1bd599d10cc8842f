#!/bin/bash
# Round artefacts in one GPU call: gpu tests, smoke, bench (cfg1 with CPU baseline, cfg4),
# reference arm, per-op profiles, launch list, UNet DRAM traffic, ncu full captures.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_cfg1.json 2> gpurun_out/bench_cfg1.err
timeout 600 python bench.py --streams 8 --n-steps 1 --guidance self_negative --no-cpu-baseline > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
timeout 300 python tools/prof_ops.py 4 > gpurun_out/prof_ops_r4.txt 2>&1
timeout 300 python tools/prof_ops.py 8 > gpurun_out/prof_ops_r8.txt 2>&1
timeout 200 python tools/taesd_prof.py 1 8 > gpurun_out/taesd_prof.txt 2>&1
timeout 200 python tools/unet_time.py 4 8 > gpurun_out/unet_time.txt 2>&1
bash tools/gpu_profile_round.sh > gpurun_out/profile_round.log 2>&1
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
timeout 600 $NCU -k 'regex:conv3x3_c64_u8|conv3x3_rgb8' -c 2 -o gpurun_out/ncu_full_taesd_head python tools/taesd_prof.py 1 > /dev/null 2>&1
tail -3 gpurun_out/pytest_gpu.log gpurun_out/smoke.log
for f in gpurun_out/bench_cfg1.json gpurun_out/bench_cfg4.json; do python tools/bench_line.py < $f; done
tail -c 600 gpurun_out/bench_reference.json
cat gpurun_out/unet_time.txt
ls gpurun_out
