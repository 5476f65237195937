# Config 1: one layer1 target, N = 8, C = 64, 56x56, fwd+bwd — per-launch
# times, CUDA-graph replay of the whole layer and the cuDNN nn.Conv2d context (TF32 off/on)
mkdir -p gpurun_out/c1
for k in seed7_k1 seed7_k0 im2col; do
  timeout 300 python scripts/kbench.py --kernel $k --batch 8 --iters 20 --json gpurun_out/c1/config1_$k.json > gpurun_out/c1/config1_$k.txt 2>&1
  head -2 gpurun_out/c1/config1_$k.txt
done
