# BASELINE config[1] (C2): Qwen3-4B geometry at 32k, adaptive budget — our arm on the B200 and the
# reference's CPU path on the same box's host cores, on the same layer, indexer and budgets.
mkdir -p gpurun_out
timeout 900 python bench.py --n 32768 --prep load --calib-margin 0.05 --steps 10 --warmup 3 > gpurun_out/c2_ours.json 2> gpurun_out/c2_ours.err
tail -c 600 gpurun_out/c2_ours.json; echo
cp bench_data/prep_distilled_n32768_h32x8_dh1024.npz gpurun_out/ 2>/dev/null
timeout 1500 python bench.py --impl reference --n 32768 --calib-margin 0.05 --ref-rows 32768 --steps 1 --warmup 0 > gpurun_out/c2_ref.json 2> gpurun_out/c2_ref.err
tail -c 1200 gpurun_out/c2_ref.json; tail -3 gpurun_out/c2_ref.err
