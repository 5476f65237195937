"""Per-kernel sampler latency at N = 20: CPU time per accepted kernel of
this package's sampler and, when /root/reference is present, of the reference's own
sampler on the same seed.  Usage: python scripts/sampler_latency.py [count]"""

import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(sampler_cls, cfg_cls, count: int) -> list:
    s = sampler_cls(cfg_cls(nodes=20, seed=0))
    out = []
    for _ in range(count):
        t = time.process_time()
        s.sample_kernel()
        out.append(time.process_time() - t)
    return out


def main() -> None:
    count = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    sys.path.insert(0, ROOT)
    from paper_2304_07741_b200.canvas.sampler import Sampler, SamplerConfig

    ts = run(Sampler, SamplerConfig, count)
    print(f"mirror:    {count} kernels, median {statistics.median(ts) * 1e3:.1f} ms, mean {statistics.mean(ts) * 1e3:.1f} ms CPU")
    ref = "/root/reference/pkg/src"
    if os.path.isdir(ref):
        for k in [k for k in sys.modules if k == "canvas" or k.startswith("canvas.")]:
            del sys.modules[k]
        sys.path.insert(0, ref)
        from canvas.sampler import Sampler as RS, SamplerConfig as RC  # noqa: E402

        ts = run(RS, RC, min(count, 15))
        print(f"reference: {min(count, 15)} kernels, median {statistics.median(ts) * 1e3:.1f} ms, mean {statistics.mean(ts) * 1e3:.1f} ms CPU")


if __name__ == "__main__":
    main()
