"""Measure the integer-pipe peaks (LOP3 / POPC / IADD lane-ops per second) on
the current GPU; these are the ALU roofline denominators that
MEASURED_PEAKS.json does not carry.  Prints one JSON line."""

from __future__ import annotations

import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_1812_10959_b200 import device as D  # noqa: E402


def main() -> None:
    D.require_cuda()
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    out = {"sm_count": sms}
    for op, name in ((0, "lop3"), (1, "popc"), (2, "iadd")):
        best = 0.0
        for threads in (256, 512, 1024):
            blocks = sms * (2048 // threads)
            D.probe_int_pipe(op, blocks, threads, 64)  # warm-up
            ops, ms = D.probe_int_pipe(op, blocks, threads, 2048)
            best = max(best, ops / (ms * 1e-3))
        out[f"{name}_lane_ops_per_s"] = best
        out[f"{name}_lanes_per_sm_clk_at_1965MHz"] = best / sms / 1.965e9
    print(json.dumps(out))


if __name__ == "__main__":
    main()
