MASTER_ADDR=127.0.0.1 MASTER_PORT=29519 RANK=0 WORLD_SIZE=1 LOCAL_RANK=0 timeout 120 python -c "
import bench, torch, torch.distributed as dist
bench.init_nccl(0, 1)
t = torch.ones(4, device='cuda'); dist.all_reduce(t); torch.cuda.synchronize()
print('{\"json\": 1}', flush=True)
dist.destroy_process_group()
" > gpurun_out/nccl_stdout.txt 2> gpurun_out/nccl_stderr.txt
echo "stdout:"; cat gpurun_out/nccl_stdout.txt; echo "stderr:"; head -5 gpurun_out/nccl_stderr.txt
