"""gemv device time vs m at fixed n (does the time step with whole waves of row blocks?).

    python scripts/gemv_msweep.py [n] > gpurun_out/gemv_msweep.json

Per m: `reps` launches in one CUDA graph over rotating copies of A (rotation > L2),
median of 5 replays."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import lift_inputs as gen  # noqa: E402
import paper_1502_02389_b200 as lift  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
    dev = torch.device("cuda:0")
    mmax = 12288
    copies = 4
    As = [gen.fill_device(torch.empty(mmax * n, device=dev), c, gen.TID_A, 0, 0, 0.0, 3.0).view(mmax, n)
          for c in range(copies)]
    gx = gen.fill_device(torch.empty(n, device=dev), 0, gen.TID_X, 0, 0, 0.0, 1.0)
    gy = gen.fill_device(torch.empty(mmax, device=dev), 0, gen.TID_Y, 0, 0, 0.0, 2.0)
    go = torch.empty(mmax, device=dev)
    out = {"n": n, "sms": torch.cuda.get_device_properties(dev).multi_processor_count}
    reps = 16
    ms = [512, 1024, 2048, 3072, 4096, 4736, 5120, 6144, 7104, 7168, 7680, 8192, 8704, 9472, 10240,
          11264, 12288]
    for m in ms:
        s = torch.cuda.Stream(device=dev)
        with torch.cuda.stream(s):
            lift.gemv(As[0][:m], gx, gy[:m], 1.5, 0.5, out=go[:m])
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                for i in range(reps):
                    lift.gemv(As[i % copies][:m], gx, gy[:m], 1.5, 0.5, out=go[:m])
            ts = []
            for _ in range(5):
                e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
                e0.record(s)
                g.replay()
                e1.record(s)
                e1.synchronize()
                ts.append(e0.elapsed_time(e1) / reps * 1e3)
        us = sorted(ts)[2]
        out[str(m)] = {"us": round(us, 2), "GB/s": round(4 * (m * n + n + 2 * m) / us / 1e3, 1)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
