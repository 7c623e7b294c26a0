"""Write-only vs copy HBM bandwidth on this B200 (context for the final pass, which is ~83%
writes): torch fill / broadcast copy of a 1 MiB random row over 2.4 GB (the cfg3 output size; fill data compresses in L2, the random row does not) and 1 GiB copies (zero / random data), CUDA events, best of 10."""
import json
import torch

def best(fn, n=10):
    ts = []
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return min(ts)

out = torch.empty(2415919104 // 4, dtype=torch.int32, device="cuda")
src = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
dst = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
for _ in range(3):
    out.fill_(1); dst.copy_(src)
torch.cuda.synchronize()
t_fill = best(lambda: out.fill_(1))
t_zero = best(lambda: out.zero_())
t_copy = best(lambda: dst.copy_(src))
row = torch.randint(0, 1 << 30, (1 << 18,), dtype=torch.int32, device="cuda")            # 1 MiB, stays in L2
o2 = out.view(-1, 1 << 18)
t_ar = best(lambda: o2.copy_(row.expand_as(o2)))
rnd = torch.randint(0, 1 << 30, (1 << 28,), dtype=torch.int32, device="cuda")           # 1 GiB of noise
src.copy_(rnd.view(torch.uint8))
t_copy_rnd = best(lambda: dst.copy_(src))
import ctypes, os
wl = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libwrite_probe.so"))
wl.write_probe.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
res_w = {}
for blocks in (148 * 4, 148 * 8, 148 * 16):
    st = torch.cuda.current_stream().cuda_stream
    wl.write_probe(out.data_ptr(), out.numel() * 4, blocks, 256, st)
    torch.cuda.synchronize()
    res_w[f"hash_write_2.4GB_gbs_{blocks}blk"] = 2415919104 / best(
        lambda: wl.write_probe(out.data_ptr(), out.numel() * 4, blocks, 256, st)) / 1e6
print(json.dumps(res_w))
print(json.dumps({"fill_2.4GB_gbs": 2415919104 / t_fill / 1e6, "zero_2.4GB_gbs": 2415919104 / t_zero / 1e6,
                  "copy_1GiB_rw_gbs": 2 * (1 << 30) / t_copy / 1e6,
                  "bcast_random_2.4GB_write_gbs": 2415919104 / t_ar / 1e6,
                  "copy_1GiB_random_rw_gbs": 2 * (1 << 30) / t_copy_rnd / 1e6}))
