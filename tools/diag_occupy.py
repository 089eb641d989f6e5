"""Lazy-loading probe for the SM-occupancy test hook (see tests/test_gpu_ffn_progress.py)."""
import sys, time, torch
sys.path.insert(0, "/root/repo")
from paper_2106_10715_b200 import device as dv
cuda = torch.device("cuda:0")
sms = torch.cuda.get_device_properties(0).multi_processor_count
release = torch.zeros(1, dtype=torch.int32, device=cuda)
timed_out = torch.zeros(1, dtype=torch.int32, device=cuda)
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
a = torch.ones(1000, device=cuda)
dv.set_flag(timed_out, stream=sb)
b = a * 2
timed_out.zero_()
torch.cuda.synchronize()
t0 = time.time()
dv.occupy_sms(sms - 4, release, timed_out, stream=sa, timeout_s=5)
with torch.cuda.stream(sb):
    b = a * 2  # preallocated? (allocation may happen)
dv.set_flag(release, stream=sb)
print("host launched", time.time() - t0, flush=True)
torch.cuda.synchronize()
print("plain kernel: timed_out", timed_out.item(), "elapsed", time.time() - t0, flush=True)
