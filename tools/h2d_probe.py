import torch, time
n = 128*500*2000
h = torch.empty(n, dtype=torch.float32).pin_memory()
h.uniform_()
d = torch.empty(n, dtype=torch.float32, device="cuda")
ss = [torch.cuda.Stream() for _ in range(4)]
def run(k, reps=10):
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        c = n // k
        for i in range(k):
            s = ss[i % len(ss)]
            s.wait_event(e0) if False else None
            with torch.cuda.stream(s):
                d[i*c:(i+1)*c].copy_(h[i*c:(i+1)*c], non_blocking=True)
        for s in ss[:k]:
            torch.cuda.current_stream().wait_stream(s)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(k, "chunks/streams:", round(ms,3), "ms", round(n*4/ms/1e6,1), "GB/s")
for k in (1, 2, 4, 1, 2, 4):
    run(k)
