# The N>1 bench path on a 1-GPU box: ranks share cuda:0, gloo for the plumbing, CPU-staged
# output assembly (VSP_BENCH_DEVICES=1 VSP_BENCH_BACKEND=gloo). Checks that every split runs
# end to end under torchrun; the NCCL assembly itself is covered by the world-1 tests.
mkdir -p gpurun_out
export VSP_BENCH_DEVICES=1 VSP_BENCH_BACKEND=gloo
CFGS=${CFGS:-"2:heads:nccl 4:heads:nccl 2:heads:mirror 4:heads:mirror 2:balanced:nccl 4:spread:nccl"}
for cfg in $CFGS; do
  IFS=: read N SH AS <<< "$cfg"
  tag=${N}_${SH}_${AS}
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29$((500 + N)) bench.py --gpus $N --shard $SH --assemble $AS --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/mr_$tag.json 2> gpurun_out/mr_$tag.err
  echo "== N=$N $SH $AS rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/mr_$tag.json')); print(d['ms_per_step'], d['config']['parallelism'][:60], d.get('assembly'), d.get('mirror_check'), d.get('allgather_ms'))" 2>/dev/null; grep -i "error\|Traceback" gpurun_out/mr_$tag.err | head -5
done
