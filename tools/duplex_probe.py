import torch, time
N = 512 << 20
h1 = torch.empty(N, dtype=torch.uint8).pin_memory(); h2 = torch.empty(N, dtype=torch.uint8).pin_memory()
d1 = torch.empty(N, dtype=torch.uint8, device='cuda'); d2 = torch.empty(N, dtype=torch.uint8, device='cuda')
s1 = torch.cuda.Stream(); s2 = torch.cuda.Stream()
def t(f):
    torch.cuda.synchronize(); t0 = time.time(); f(); torch.cuda.synchronize(); return (time.time() - t0) * 1e3
for _ in range(2):
    a = t(lambda: h1.copy_(d1, non_blocking=True))
    b = t(lambda: d2.copy_(h2, non_blocking=True))
    def both():
        with torch.cuda.stream(s1): h1.copy_(d1, non_blocking=True)
        with torch.cuda.stream(s2): d2.copy_(h2, non_blocking=True)
    c = t(both)
    print(f"D2H {a:.2f} ms ({N/a/1e6:.1f} GB/s)  H2D {b:.2f} ms ({N/b/1e6:.1f} GB/s)  both {c:.2f} ms")
print(torch.cuda.get_device_properties(0))
import subprocess; print(subprocess.run(["nvidia-smi", "-q", "-d", "PCI"], capture_output=True, text=True).stdout[:1500])
