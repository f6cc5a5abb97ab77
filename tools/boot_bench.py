"""One-GPU bootstrap latency outside the full bench: python tools/boot_bench.py"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402


def main():
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)

    def t_ms(fn, reps=5):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return statistics.median(ts)
    print(json.dumps(bench.bootstrap_bench(stream, t_ms)))
    for B in [int(b) for b in os.environ.get("SECPE_N4_BATCHES", "8").split(",")]:
        print(json.dumps(bench.argmax_k16_bench(stream, t_ms, B)))
    print(json.dumps(bench.argmax_boot_bench(stream, t_ms, "argmax_n256", 8, 6.0)))
    print(json.dumps(bench.clip_bench(stream, t_ms)))


if __name__ == "__main__":
    main()
