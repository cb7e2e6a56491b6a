mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --backend gloo --share-gpu > gpurun_out/mr2.json 2> gpurun_out/mr2.err; echo "multirank exit $?"
cat gpurun_out/mr2.json | cut -c1-1500; tail -5 gpurun_out/mr2.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 --ref-seconds 3 > gpurun_out/ref.json 2> gpurun_out/ref.err; echo "ref exit $?"
cat gpurun_out/ref.json; tail -3 gpurun_out/ref.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 2 --steps 1 --warmup 1 --ref-seconds 2 > gpurun_out/ref2.json 2> gpurun_out/ref2.err; echo "ref2 exit $?"; cat gpurun_out/ref2.json | cut -c1-300
