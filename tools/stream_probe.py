"""Weight-streaming probe (include/hs_probes.h hs_debug_stream_probe): GB/s of the decode stack's
TMA pattern over the image's row-major layout vs a tiled (contiguous 16 KiB block) layout."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402,F401

from paper_2502_15524_b200 import hs  # noqa: E402

out = []
for M, K in ((65536, 4096), (131072, 4096)):  # 512 MB / 1 GB: larger than L2
    for slots in (8, 12):
        for layout in (0, 1, 2, 3):
            out.append(dict(M=M, K=K, slots=slots, layout=["row-major", "tiled", "row-major+mma", "tiled+mma"][layout],
                            gbs=round(hs.stream_probe(layout, M, K, slots, 2), 1)))
            print(json.dumps(out[-1]), flush=True)
