# Strong-scaling run of the bench over 1, 2, 4, 8 GPUs of one node (the
# driver's SCALE protocol): one torchrun per N, NCCL all-reduce of the counts.
#   CONFIG=c2 bash tools/scale.sh        (C2: M = 1e9, n = 50, N = 500)
#   CONFIG=c5 PATHS=4e9 bash tools/scale.sh   (C5 at its BASELINE M = 4e9)
CONFIG=${CONFIG:-c2}
EXTRA=${PATHS:+--paths $PATHS}
mkdir -p gpurun_out
for N in ${NS:-1 2 4 8}; do
  if [ "$N" -gt "$(nvidia-smi -L | wc -l)" ]; then echo "skip N=$N (fewer GPUs)"; continue; fi
  if [ "$N" = 1 ]; then
    python bench.py --config $CONFIG $EXTRA --no-cpu-baseline
  else
    NCCL_DEBUG=INFO python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
      --master-addr 127.0.0.1 --master-port $((29500 + N)) bench.py --gpus $N --config $CONFIG $EXTRA \
      2> gpurun_out/scale_${CONFIG}_n${N}.err
  fi
done | tee gpurun_out/scale_${CONFIG}.jsonl
