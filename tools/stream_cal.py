"""HBM streaming calibration: LDG.128 vs cp.async.bulk rings (profiles/r1_gram_tc.md)."""
import ctypes as C, torch
import os
# build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC -o tools/stream_cal.so tools/stream_cal.cu
lib = C.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "stream_cal.so"))
lib.run_ldg.restype = C.c_float; lib.run_bulk.restype = C.c_float
nbytes = 18_560_000_000
x = torch.empty(nbytes // 4, dtype=torch.float32, device='cuda').uniform_()
out = torch.zeros(4, device='cuda'); torch.cuda.synchronize()
X, O = C.c_void_p(x.data_ptr()), C.c_void_p(out.data_ptr())
for g, bl in [(148*4, 512), (148*8, 256), (148*16, 256)]:
    ms = lib.run_ldg(X, C.c_long(nbytes), O, g, bl, 3); print(f"ldg grid {g}x{bl}: {ms:.2f} ms {nbytes/ms/1e6:.0f} GB/s", flush=True)
for chunk, NS in [(14848, 8), (14848, 12), (7424, 16), (29696, 6), (4096, 32), (16384, 12)]:
    for grid in [148, 296]:
        if grid == 296 and chunk * NS > 110000: continue
        ms = lib.run_bulk(X, C.c_long(nbytes), O, chunk, NS, grid, 3)
        print(f"bulk chunk {chunk} NS {NS} grid {grid}: {ms:.2f} ms {nbytes/ms/1e6:.0f} GB/s  inflight/SM {chunk*NS*grid/148/1024:.0f} KB", flush=True)
