nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv,noheader -lms 50 > gpurun_out/clk.csv &
SMI=$!
python -c "
import torch; p=torch.cuda.get_device_properties(0); print('uuid', getattr(p,'uuid',None))
a=torch.randn(8192,8192,device='cuda',dtype=torch.bfloat16)
import time; t=time.time()
while time.time()-t<2: a@a
torch.cuda.synchronize()
"
timeout 300 python tools/profile_kernels.py --batch 1 --plans FULLY_QUANT:12 2>&1 | tail -9
kill $SMI
awk -F, '{print $1}' gpurun_out/clk.csv | sort | uniq -c | sort -rn | head -8
