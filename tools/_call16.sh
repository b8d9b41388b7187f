set -x
for m in fp32 tf32; do for b in 256 32 1; do CONV2D_FORCE_WINO_VARIANT=1 timeout 600 python bench_layers.py --set R4,R10,R17,R24,V2,V4,V6,V8 --batch $b --math $m --algos winograd_f2x2_3x3 --iters 5 --warmup 2 --out gpurun_out/r2_wf_b${b}_${m}.json > gpurun_out/r2_wf_b${b}_${m}.log 2>&1; done; done
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/r2_plain_step.log 2>&1 && ncu --nvtx --nvtx-include "bench_timed/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_step_launches.csv $CMD > gpurun_out/r2_ncu_step.log 2>&1
CMD2="python bench_layers.py --set R4 --batch 256 --algos implicit_gemm --iters 2 --warmup 1"
$CMD2 > gpurun_out/r2_plain_r4.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:halo -s 2 -c 1 -o gpurun_out/r2_r4_halo $CMD2 > gpurun_out/r2_ncu_r4.log 2>&1
echo finished
