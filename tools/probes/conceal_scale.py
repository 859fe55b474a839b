"""conceal_image at image scale with the reference's CLI defaults (dft, 250
iterations) in block mode: wall time per call and per block, report sanity."""
import sys
import time

import numpy as np

from paper_2204_14194_b200 import conceal_image

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
spec = sys.argv[2] if len(sys.argv) > 2 else "dft"
rng = np.random.default_rng(5)
yy, xx = np.mgrid[0:n, 0:n]
img = np.clip(128 + 50 * np.sin(0.05 * yy + 0.03 * xx) + 30 * np.cos(0.11 * xx) + rng.normal(0, 4, (n, n)), 0, 255)
img = np.rint(img)
tiles = [(r, c) for r in range(0, n, 16) for c in range(0, n, 16)]
pick = rng.choice(len(tiles), len(tiles) // 10, replace=False)
lost = np.zeros((n, n), dtype=bool)
for i in pick:
    r, c = tiles[i]
    lost[r:r + 16, c:c + 16] = True
obs = img.copy()
obs[lost] = 0
for rep in range(2):
    t0 = time.perf_counter()
    out, report = conceal_image(obs, lost, dict_spec=spec, block=(16, 16), reference=img, device="cuda:0")
    dt = time.perf_counter() - t0
    print(f"{n}x{n} {spec}: {len(report['blocks'])} blocks in {dt:.2f} s "
          f"({dt / max(1, len(report['blocks'])) * 1e3:.1f} ms/block), PSNR {report['psnr_db']:.2f} dB")
