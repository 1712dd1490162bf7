mkdir -p gpurun_out
python bench.py --steps 5 --warmup 3 > gpurun_out/drv_n1.json 2> gpurun_out/drv_n1.err
for n in 2 4; do
python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600+n)) bench.py --gpus $n --steps 5 --warmup 3 > gpurun_out/drv_n$n.json 2> gpurun_out/drv_n$n.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29700+n)) bench.py --impl reference --gpus $n --steps 2 --warmup 1 > gpurun_out/drv_ref_n$n.json 2> gpurun_out/drv_ref_n$n.err
done
for f in gpurun_out/drv_*.json; do echo "$f: $(python -c "import json,sys;d=json.load(open('$f'));print(d.get('value'),d.get('n_gpus'),(d.get('e2e') or {}).get('value'),d.get('ms_per_step'))" 2>&1)"; done
