#!/bin/bash
# Round measurement set: config-1 leg, per-layer oracle leg, the Fig.-1 per-layer
# tables (every algorithm, ResNet-50 b1/b32/b256 and VGG-16 b1/b32, both math modes) and the stack's
# auto-selected per-layer tables at b256 / b32, the fused-Winograd tables, and (--ncu) the timed-step ncu launch
# list plus full captures of the R4 (3x3 halo) and V1 (4-channel halo) kernels.  Output: gpurun_out/r2_*.
set -x
python bench.py --config1 > gpurun_out/r2_config1.json 2> gpurun_out/r2_config1.err
python bench.py --oracle-layers > gpurun_out/r2_oracle_layers.json 2> gpurun_out/r2_oracle_layers.err
for m in fp32 tf32; do
  for b in 1 32 256; do timeout 900 python bench_layers.py --set resnet50 --batch $b --math $m --iters 5 --warmup 2 --out gpurun_out/r2_tab_resnet50_b${b}_${m}.json > gpurun_out/r2_tab_resnet50_b${b}_${m}.log 2>&1; done
  for b in 1 32; do timeout 900 python bench_layers.py --set vgg16 --batch $b --math $m --iters 5 --warmup 2 --out gpurun_out/r2_tab_vgg16_b${b}_${m}.json > gpurun_out/r2_tab_vgg16_b${b}_${m}.log 2>&1; done
done
for b in 256 32; do timeout 900 python bench_layers.py --set stack --batch $b --algos auto --iters 5 --warmup 2 --out gpurun_out/r2_stack_auto_b${b}.json > gpurun_out/r2_stack_auto_b${b}.log 2>&1; done
for m in fp32 tf32; do for b in 256 32 1; do CONV2D_FORCE_WINO_VARIANT=1 timeout 600 python bench_layers.py --set R4,R10,R17,R24,V2,V4,V6,V8 --batch $b --math $m --algos winograd_f2x2_3x3 --iters 5 --warmup 2 --out gpurun_out/r2_wf_b${b}_${m}.json > gpurun_out/r2_wf_b${b}_${m}.log 2>&1; done; done
if [ "$1" = "--ncu" ]; then
  # each capture only after its own command has exited 0 without ncu
  CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
  $CMD > gpurun_out/r2_plain_step.log 2>&1 && ncu --nvtx --nvtx-include "bench_timed/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_step_launches.csv $CMD > gpurun_out/r2_ncu_step.log 2>&1
  CMD2="python bench_layers.py --set R4 --batch 256 --algos implicit_gemm --iters 2 --warmup 1"
  $CMD2 > gpurun_out/r2_plain_r4.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:halo -s 2 -c 1 -o gpurun_out/r2_r4_halo -f $CMD2 > gpurun_out/r2_ncu_r4.log 2>&1
  CMD3="python bench_layers.py --set V1 --batch 32 --algos implicit_gemm --iters 2 --warmup 1"
  $CMD3 > gpurun_out/r2_plain_v1.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:halo -s 2 -c 1 -o gpurun_out/r2_v1_c4 -f $CMD3 > gpurun_out/r2_ncu_v1.log 2>&1
fi
echo finished
