"""Pinned host <-> device copy bandwidth: contiguous vs the head-chunked 2-D
copies the host-buffer layer issues (Wan: 40 heads x 128 x bf16 rows)."""
import torch, ctypes
cudart = ctypes.CDLL("libcudart.so")
S, H, d = 75600, 40, 128
x = torch.empty((S, H, d), dtype=torch.bfloat16).pin_memory()
y = torch.empty((S, H, d), dtype=torch.bfloat16, device="cuda")
st = torch.cuda.Stream()
nbytes = x.numel() * 2
def timed(fn, reps=5):
    fn(); st.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(st)
    for _ in range(reps): fn()
    e1.record(st); st.synchronize()
    return e0.elapsed_time(e1) / reps
def contig():
    with torch.cuda.stream(st): y.copy_(x, non_blocking=True)
row = H * d * 2
def chunked(heads_per):
    def f():
        for h0 in range(0, H, heads_per):
            w = min(heads_per, H - h0) * d * 2
            off = h0 * d * 2
            r = cudart.cudaMemcpy2DAsync(ctypes.c_void_p(y.data_ptr() + off), ctypes.c_size_t(row),
                                         ctypes.c_void_p(x.data_ptr() + off), ctypes.c_size_t(row),
                                         ctypes.c_size_t(w), ctypes.c_size_t(S), 1, ctypes.c_void_p(st.cuda_stream))
            assert r == 0, r
    return f
t = timed(contig); print(f"H2D contiguous {nbytes/1e9:.2f} GB {t:.2f} ms {nbytes/t/1e6:.1f} GB/s")
for hp in (1, 2, 5, 10, 20, 40):
    t = timed(chunked(hp)); print(f"H2D 2D chunks of {hp} heads ({hp*d*2} B rows) {t:.2f} ms {nbytes/t/1e6:.1f} GB/s")
def d2h():
    with torch.cuda.stream(st): x.copy_(y, non_blocking=True)
t = timed(d2h); print(f"D2H contiguous {t:.2f} ms {nbytes/t/1e6:.1f} GB/s")
# two H2D streams in parallel (halves of the tensor)
st2 = torch.cuda.Stream()
half = S // 2
def two():
    with torch.cuda.stream(st):
        y[:half].copy_(x[:half], non_blocking=True)
    with torch.cuda.stream(st2):
        y[half:].copy_(x[half:], non_blocking=True)
def timed2(fn, reps=5):
    fn(); torch.cuda.synchronize()
    import time
    t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3 / reps
t = timed2(two); print(f"H2D two streams {t:.2f} ms {nbytes/t/1e6:.1f} GB/s")
t = timed2(contig); print(f"H2D one stream (wall) {t:.2f} ms {nbytes/t/1e6:.1f} GB/s")
