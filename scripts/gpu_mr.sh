# Multi-rank dry run of the torchrun path on a one-GPU box (both ranks pinned
# to GPU 0 via SCZ_BENCH_DEVICE, gloo for barrier/reductions), weak and strong
# scaling, plus the reference arm under torchrun; then compute-sanitizer
# racecheck over the v2 / batch / search parity tests.
mkdir -p gpurun_out
export SCZ_BENCH_DEVICE=0
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 2 --steps 10 --warmup 3 --no-extras --no-cpu-baseline --no-configs > gpurun_out/mr_weak.json 2> gpurun_out/mr_weak.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --gpus 2 --steps 5 --warmup 3 --workload resnet50 --global-batch 4096 --no-extras --no-cpu-baseline --no-configs --no-e2e > gpurun_out/mr_strong.json 2> gpurun_out/mr_strong.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 \
  bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > gpurun_out/mr_ref.json 2> gpurun_out/mr_ref.err
unset SCZ_BENCH_DEVICE
timeout 2400 compute-sanitizer --tool racecheck --error-exitcode 17 --target-processes all \
  python -m pytest tests -m gpu -x -q -p no:cacheprovider \
  -k "v2_containers_match_oracle or lanes_are_reference or batch_api or lazy_search or device_header_decode_matches or mixed_symbol or heterogeneous or random_round_trips" \
  > gpurun_out/sanitize_racecheck.log 2>&1
echo "racecheck rc=$?" >> gpurun_out/sanitize_racecheck.log
