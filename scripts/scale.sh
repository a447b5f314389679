# Multi-GPU scaling runs for an 8-GPU B200 node (not runnable on the
# single-GPU pool this build was developed on).  One process per GPU over
# NCCL; every line is the driver's contract line (max-over-ranks device time).
#   C5 weak (default: one 16384^2 strip per rank), C5 and C3 strong, C4 strong,
#   and the device-collective variants.
run() { local n=$1; shift
  if [ $n = 1 ]; then python bench.py --gpus 1 --steps 20 --warmup 5 "$@"
  else python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
       --master-port $((29500 + n)) bench.py --gpus $n --steps 20 --warmup 5 "$@"; fi; }
mkdir -p gpurun_out/scale
for n in 1 2 4 8; do
  run $n > gpurun_out/scale/c5_weak_$n.json
  run $n --config c5 --strong --force-sharded > gpurun_out/scale/c5_strong_$n.json
  run $n --config c3 --strong --force-sharded > gpurun_out/scale/c3_strong_$n.json
  run $n --config c4 --strong --force-sharded > gpurun_out/scale/c4_strong_$n.json
  run $n --device-halo --force-sharded > gpurun_out/scale/c5_weak_devhalo_$n.json
done
