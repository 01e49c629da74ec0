set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/clocks_dmma.csv &
SMI=$!
./build/dmma_peak | tee gpurun_out/dmma_peak.json
python -c "
import torch,time
a=torch.randn(8192,8192,dtype=torch.float64,device='cuda'); b=torch.randn(8192,8192,dtype=torch.float64,device='cuda')
for _ in range(2): c=a@b
torch.cuda.synchronize()
e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
best=1e9
for _ in range(5):
  e0.record(); c=a@b; e1.record(); torch.cuda.synchronize(); best=min(best,e0.elapsed_time(e1))
print('torch_dgemm_8192_tflops', 2*8192**3/(best*1e-3)/1e12)
" | tee gpurun_out/torch_dgemm.txt
kill $SMI
