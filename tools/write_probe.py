import sys, torch
sys.path.insert(0, "tools")
import membench
L = membench.build()
sms = torch.cuda.get_device_properties(0).multi_processor_count
n = 1 << 30
dst = torch.empty(n // 4, dtype=torch.float32, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for _ in range(2):
    L.mb_write(dst.data_ptr(), n, sms * 64, 256, 1, 4, s)
    L.mb_write_os(dst.data_ptr(), n, 32, 256, 2, s)
torch.cuda.synchronize()
