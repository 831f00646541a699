bash tools/gpu_round.sh
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
BLEST_DIST_BACKEND=gloo timeout 600 $T --master-port 29511 bench.py --gpus 2 --config c1 --steps 4 --warmup 3 > gpurun_out/m_rep.json 2> gpurun_out/m_rep.err
BLEST_DIST_BACKEND=gloo timeout 600 $T --master-port 29512 bench.py --gpus 2 --config c1 --steps 4 --warmup 3 --partition rows > gpurun_out/m_rows.json 2> gpurun_out/m_rows.err
timeout 600 $T --master-port 29513 bench.py --gpus 2 --config c1 --steps 4 --warmup 3 --impl reference > gpurun_out/m_ref.json 2> gpurun_out/m_ref.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29514 bench.py --gpus 1 --config c1 --steps 4 --warmup 3 > gpurun_out/m_one.json 2> gpurun_out/m_one.err
