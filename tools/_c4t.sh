cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; exec > gpurun_out/c4t.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guard.py -x -q -k "c4 or guard or config1" 2>&1 | tail -3
timeout 900 python tools/fuzz_gpu.py --cases 300 --seed 9 --focus c4 | tail -5
for m in 0 1; do for b in 32 8 1; do
 timeout 120 python tools/time_layer.py $b 224 224 3 64 3 3 1 1 0 $m 2>&1 | tail -1
done; done
