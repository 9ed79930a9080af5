#!/bin/bash
# Functional test of bench.py's N > 1 path (two ranks, gloo, both on cuda:0;
# not a measurement): weak and strong scaling lines must parse and count
# both ranks' systems.
export NLK_BENCH_DEVICE=0 NLK_BENCH_BACKEND=gloo
for mode in "--batch 65536" "--global-batch 100000"; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 \
    bench.py --gpus 2 --config c4 $mode --steps 2 --warmup 1 --e2e-steps 1 > gpurun_out/torchrun2.json 2> gpurun_out/torchrun2.err
  echo "rc=$?"
  python -c "
import json; d=json.load(open('gpurun_out/torchrun2.json')); print(d['n_gpus'], d['scaling'], d['config']['global_batch_per_job'], d['config']['systems_per_step_per_gpu'], round(d['value']/1e6,2), 'e2e', round(d['e2e']['value']/1e6,2), d.get('parity'))"
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29518 \
    bench.py --impl reference --gpus 2 --config c4 --steps 1 --warmup 0 --cpu-sample 20 > gpurun_out/torchrun2_ref.json 2>> gpurun_out/torchrun2.err
echo "ref rc=$?"; head -c 300 gpurun_out/torchrun2_ref.json; echo
