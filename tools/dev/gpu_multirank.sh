# The N>1 bench path on a 1-GPU box: ranks share cuda:0, gloo for the plumbing, CPU-staged
# output assembly (VSP_BENCH_DEVICES=1 VSP_BENCH_BACKEND=gloo). Checks that every split runs
# end to end under torchrun; the NCCL assembly itself is covered by the world-1 tests.
mkdir -p gpurun_out
export VSP_BENCH_DEVICES=1 VSP_BENCH_BACKEND=gloo
for cfg in "2 heads" "4 heads" "2 balanced" "4 spread"; do
  set -- $cfg
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port 29$((500 + $1)) bench.py --gpus $1 --shard $2 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/mr_$1_$2.json 2> gpurun_out/mr_$1_$2.err
  echo "== N=$1 $2 rc=$?"; tail -c 300 gpurun_out/mr_$1_$2.json; echo; grep -i "error\|Traceback" gpurun_out/mr_$1_$2.err | head -5
done
