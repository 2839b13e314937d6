import ctypes as C, zlib, numpy as np, sys, time
lib = C.CDLL("/root/repo/tests/native/libzmodel.so")
lib.zmodel_compress.argtypes=[C.c_char_p, C.c_uint64, C.c_int, C.c_char_p, C.c_uint64, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
def model(data, chunk=4096):
    cap = len(data)*2+1024
    out = C.create_string_buffer(cap); ol = C.c_uint64(); st=(C.c_uint64*6)()
    rc = lib.zmodel_compress(data, len(data), chunk, out, cap, C.byref(ol), st)
    assert rc == 0, rc
    return out.raw[:ol.value], list(st)
def check(data, name, chunk=4096):
    a, st = model(data, chunk); b = zlib.compress(data, 6)
    ok = a == b
    if not ok:
        i = next((i for i in range(min(len(a),len(b))) if a[i]!=b[i]), min(len(a),len(b)))
        print("FAIL", name, len(data), len(a), len(b), "first diff", i, st)
    return ok
rng = np.random.default_rng(0)
bad = 0; tot = 0
def gen():
    yield "zeros1", bytes(1)
    yield "zeros3", bytes(3)
    for n in [1,2,3,4,5,10,100,1000,4095,16383,16384,40000,65535,65536,65537,65800,70000,100000,200000,300000]:
        yield f"zeros{n}", bytes(n)
        yield f"rand{n}", rng.integers(0,256,n,dtype=np.uint8).tobytes()
        for p in (0.01, 0.1, 0.3, 0.5):
            bits = (rng.random(n*8) < p).astype(np.uint8)
            yield f"bits{p}_{n}", np.packbits(bits, bitorder='little').tobytes()
        yield f"text{n}", (b"the quick brown fox jumps over the lazy dog %d " * (n//40+1))[:n]
        yield f"small_alpha{n}", rng.integers(0,4,n,dtype=np.uint8).tobytes()
        yield f"runs{n}", np.repeat(rng.integers(0,3,n//50+1,dtype=np.uint8), rng.integers(1,300,n//50+1))[:n].tobytes()
for name, data in gen():
    tot += 1
    if not check(data, name): bad += 1
    if not check(data, name+"_ch257", 257): bad += 1
print("total", tot, "bad", bad)
