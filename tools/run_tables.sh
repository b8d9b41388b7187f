set -x
for m in fp32 tf32; do
  for b in 1 32 256; do python bench_layers.py --set resnet50 --batch $b --math $m --iters 5 --warmup 2 --out gpurun_out/tab_resnet50_b${b}_${m}.json > gpurun_out/tab_resnet50_b${b}_${m}.log 2>&1; done
  for b in 1 32; do python bench_layers.py --set vgg16 --batch $b --math $m --iters 5 --warmup 2 --out gpurun_out/tab_vgg16_b${b}_${m}.json > gpurun_out/tab_vgg16_b${b}_${m}.log 2>&1; done
done
