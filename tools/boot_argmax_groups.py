import os, sys, json, statistics
sys.path.insert(0, "/root/repo")
import torch, bench
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream)
def t_ms(fn, reps=3):
    for _ in range(1): fn()
    torch.cuda.synchronize(); ts=[]
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream); fn(); b.record(stream); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return statistics.median(ts)
for pn, g in (("boot_argmax16", (4, 5, 6)), ("boot_argmax16_g4", (3, 4, 4, 4)), ("boot_argmax16_g4", (4, 4, 4, 3))):
    r = bench.argmax_boot_bench(stream, t_ms, "argmax_k16", 8, 2.0, pn, g)
    print(pn, g, round(r["query_argmax_per_s"], 1), r["labels_exact_above_margin"], flush=True)
