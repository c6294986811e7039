#!/bin/bash
# bench.py under torchrun with 2 and 4 ranks on the one available GPU (ranks share the device:
# exercises the launch path, slab split, IPC linking and the max-over-ranks reduction the
# driver's N>1 runs use; numbers are not multi-GPU numbers).
mkdir -p gpurun_out
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29600 + n)) bench.py --gpus $n --allow-shared-gpu --steps 100 --warmup 5 --sweep-steps 50 --e2e-reps 2 \
      > gpurun_out/mr_bench_$n.json 2> gpurun_out/mr_bench_$n.err
  echo "ours N=$n rc=$?"; tail -c 1500 gpurun_out/mr_bench_$n.json; echo
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29610 + n)) bench.py --impl reference --gpus $n --steps 2 --warmup 3 \
      > gpurun_out/mr_ref_$n.json 2> gpurun_out/mr_ref_$n.err
  echo "reference N=$n rc=$?"; cat gpurun_out/mr_ref_$n.json; echo
done
