import time, numpy as np, torch
n = 1914884608 // 8
x = torch.randn(n, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
def t(name, fn, reps=2):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    print(f"{name}: {(time.perf_counter() - t0) / reps * 1e3:.1f} ms", flush=True)
t("cpu()", lambda: x.cpu().numpy())
stage = torch.empty(64 * 1024 * 1024 // 8, dtype=torch.float64, pin_memory=True)
def staged():
    out = np.empty(n, dtype=np.float64)
    ch = stage.numel()
    sv = stage.numpy()
    for i in range(0, n, ch):
        m = min(ch, n - i)
        stage[:m].copy_(x[i:i + m], non_blocking=False)
        out[i:i + m] = sv[:m]
    return out
t("staged 64MB", staged)
def pinned_alloc():
    p = torch.empty(n, dtype=torch.float64, pin_memory=True)
    p.copy_(x)
    return p.numpy()
t("pin alloc + copy", pinned_alloc)
st2 = [torch.empty(64 * 1024 * 1024 // 8, dtype=torch.float64, pin_memory=True) for _ in range(2)]
s2 = torch.cuda.Stream()
def staged2():
    out = np.empty(n, dtype=np.float64)
    ch = st2[0].numel()
    evs = [torch.cuda.Event(), torch.cuda.Event()]
    chunks = list(range(0, n, ch))
    def issue(k):
        i = chunks[k]; m = min(ch, n - i)
        with torch.cuda.stream(s2):
            st2[k % 2][:m].copy_(x[i:i + m], non_blocking=True)
            evs[k % 2].record(s2)
    issue(0)
    for k in range(len(chunks)):
        if k + 1 < len(chunks): issue(k + 1)
        evs[k % 2].synchronize()
        i = chunks[k]; m = min(ch, n - i)
        out[i:i + m] = st2[k % 2].numpy()[:m]
    return out
t("double-buffered 64MB", staged2)
