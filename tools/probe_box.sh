mkdir -p gpurun_out
{
nvidia-smi
nvidia-smi topo -m
nvidia-smi -q | grep -i -A3 -E "pci|link" | head -80
nvidia-smi nvlink -s 2>&1 | head -40
echo CUDA_VISIBLE_DEVICES=$CUDA_VISIBLE_DEVICES
nproc; lscpu | head -30; numactl -H 2>&1 | head; free -g
python -c "import torch; print('ndev', torch.cuda.device_count(), torch.cuda.get_device_name(0)); p=torch.cuda.get_device_properties(0); print(p)"
python - <<'PY'
import torch, time
torch.cuda.init()
a=torch.empty(512<<20, dtype=torch.uint8, device='cuda')
h=torch.empty(512<<20, dtype=torch.uint8, pin_memory=True)
for name, f in [('d2h', lambda: h.copy_(a, non_blocking=True)), ('h2d', lambda: a.copy_(h, non_blocking=True))]:
    for _ in range(2): f()
    torch.cuda.synchronize()
    s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
    s.record(); 
    for _ in range(5): f()
    e.record(); torch.cuda.synchronize()
    print(name, 5*a.numel()/(s.elapsed_time(e)*1e-3)/1e9, 'GB/s')
b=torch.empty_like(a)
for _ in range(3): b.copy_(a)
s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); s.record()
for _ in range(10): b.copy_(a)
e.record(); torch.cuda.synchronize()
print('d2d copy delivered', 10*a.numel()/(s.elapsed_time(e)*1e-3)/1e9, 'GB/s')
PY
} > gpurun_out/probe.txt 2>&1
