#!/bin/bash
# Round measurement set: config-1 leg, per-layer oracle leg, the Fig.-1 per-layer
# tables (every algorithm, ResNet-50 b1/b32/b256 and VGG-16 b1/b32, both math modes) and the stack's
# auto-selected per-layer tables at b256 / b32.  Output: gpurun_out/r2_*.
set -x
python bench.py --config1 > gpurun_out/r2_config1.json 2> gpurun_out/r2_config1.err
python bench.py --oracle-layers > gpurun_out/r2_oracle_layers.json 2> gpurun_out/r2_oracle_layers.err
for m in fp32 tf32; do
  for b in 1 32 256; do timeout 900 python bench_layers.py --set resnet50 --batch $b --math $m --iters 5 --warmup 2 --out gpurun_out/r2_tab_resnet50_b${b}_${m}.json > gpurun_out/r2_tab_resnet50_b${b}_${m}.log 2>&1; done
  for b in 1 32; do timeout 900 python bench_layers.py --set vgg16 --batch $b --math $m --iters 5 --warmup 2 --out gpurun_out/r2_tab_vgg16_b${b}_${m}.json > gpurun_out/r2_tab_vgg16_b${b}_${m}.log 2>&1; done
done
for b in 256 32; do timeout 900 python bench_layers.py --set stack --batch $b --algos auto --iters 5 --warmup 2 --out gpurun_out/r2_stack_auto_b${b}.json > gpurun_out/r2_stack_auto_b${b}.log 2>&1; done
