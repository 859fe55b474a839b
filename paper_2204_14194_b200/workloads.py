"""Seeded synthetic inputs for the five BASELINE configurations.

BASELINE.json describes the configs in prose and leaves generator details open;
the choices made here are fixed
in this one module, which the GPU path, the oracle tests, the golden-fixture
script and the CPU baseline all use, so every consumer sees bit-identical
inputs. There is no public dataset: every input is synthetic.

Seeding follows the reference's harness convention ``default_rng([seed, t])``
(``pkg/src/fase/verify.py:111``): block b of config c draws from
``default_rng([c, b])``; frames draw from ``default_rng([c, 1_000_000])``.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .dictionary import Dictionary, parse_dict_spec
from .grid import ExtrapConfig

FRAME_SEED = 1_000_000
GAUSS_SEED = 2204


@dataclass(frozen=True)
class Workload:
    """One BASELINE config made concrete."""

    cid: int
    name: str
    area: tuple[int, int]
    dict_spec: str
    n_atoms: int
    config: ExtrapConfig
    n_blocks: int = 1
    loss: tuple[int, int] | None = None          # centred loss (shared-geometry configs)
    frame: tuple[int, int] | None = None         # (height, width) for frame configs
    macroblock: int = 0
    loss_fraction: float = 0.0
    support: int = 0
    notes: dict = field(default_factory=dict)

    @property
    def shared_geometry(self) -> bool:
        return self.frame is None

    def dictionary(self) -> Dictionary:
        return parse_dict_spec(self.dict_spec, *self.area)


WORKLOADS = {
    0: Workload(0, "c0-single-dct48", (48, 48), "dct", 2304, ExtrapConfig(100, 0.5, 0.8),
                n_blocks=1, loss=(16, 16)),
    1: Workload(1, "c1-batch1024-dct+had48", (48, 48), "union:dct+had", 4608,
                ExtrapConfig(200, 0.5, 0.8), n_blocks=1024, loss=(16, 16)),
    2: Workload(2, "c2-frame1080p-dct+had48", (48, 48), "union:dct+had", 4608,
                ExtrapConfig(200, 0.5, 0.8), frame=(1080, 1920), macroblock=16,
                loss_fraction=0.10, support=16),
    3: Workload(3, "c3-frame2160p-rdft+brdft32", (32, 32), "union:rdft+brdft", 2048,
                ExtrapConfig(150, 0.5, 0.8), frame=(2160, 3840), macroblock=8,
                loss_fraction=0.20, support=12),
    4: Workload(4, "c4-gauss8192-64x64", (64, 64), f"gauss:8192:{GAUSS_SEED}", 8192,
                ExtrapConfig(500, 0.5, 0.85), n_blocks=4096, loss=(24, 24)),
}


def central_loss_mask(m_rows: int, n_cols: int, loss_rows: int, loss_cols: int) -> np.ndarray:
    """Centred loss block at ((M-l)//2, (N-l)//2) (``pkg/src/fase/verify.py:37-49``)."""
    if not (1 <= loss_rows <= m_rows and 1 <= loss_cols <= n_cols):
        from .errors import ParameterError
        raise ParameterError(f"loss block {loss_rows}x{loss_cols} does not fit {m_rows}x{n_cols}")
    if loss_rows == m_rows and loss_cols == n_cols:
        from .errors import ParameterError
        raise ParameterError("loss block covers the whole area; no support left")
    mask = np.zeros((m_rows, n_cols), dtype=bool)
    r0 = (m_rows - loss_rows) // 2
    c0 = (n_cols - loss_cols) // 2
    mask[r0:r0 + loss_rows, c0:c0 + loss_cols] = True
    return mask


def cosine_signal(rng: np.random.Generator, m_rows: int, n_cols: int) -> np.ndarray:
    """128 + sum of 8 random 2-D cosines + N(0, 2^2), clipped to [0, 255].

    Frequencies U[0, pi], amplitudes U[0, 40], phases U[0, 2pi) (the phase is
    unspecified in BASELINE; U[0, 2pi) is the Appendix-A choice).
    """
    wm = rng.uniform(0.0, np.pi, 8)
    wn = rng.uniform(0.0, np.pi, 8)
    amp = rng.uniform(0.0, 40.0, 8)
    ph = rng.uniform(0.0, 2.0 * np.pi, 8)
    noise = rng.normal(0.0, 2.0, (m_rows, n_cols))
    m = np.arange(m_rows, dtype=np.float64)[:, None]
    n = np.arange(n_cols, dtype=np.float64)[None, :]
    s = np.full((m_rows, n_cols), 128.0)
    for i in range(8):
        s = s + amp[i] * np.cos(wm[i] * m + wn[i] * n + ph[i])
    return np.clip(s + noise, 0.0, 255.0)


def block_signals(cid: int, n_blocks: int, m_rows: int, n_cols: int, first: int = 0) -> np.ndarray:
    """(n_blocks, M, N) float64 signals, block b from ``default_rng([cid, first + b])``."""
    out = np.empty((n_blocks, m_rows, n_cols), dtype=np.float64)
    for b in range(n_blocks):
        out[b] = cosine_signal(np.random.default_rng([cid, first + b]), m_rows, n_cols)
    return out


# ----------------------------------------------------------------- frames


def texture_frame(rng: np.random.Generator, height: int, width: int) -> np.ndarray:
    """Config-2 luma: 64 oriented sinusoids plus 1/f noise, uint8.

    f ~ U[1/64, 1/4] cycles/px, theta ~ U[0, pi), a ~ U[0, 16], phase U[0, 2pi);
    noise: white Gaussian shaped by 1/|f| in the rfft2 domain, scaled to std 8.
    """
    y = np.arange(height, dtype=np.float64)[:, None]
    x = np.arange(width, dtype=np.float64)[None, :]
    f = rng.uniform(1.0 / 64.0, 0.25, 64)
    th = rng.uniform(0.0, np.pi, 64)
    amp = rng.uniform(0.0, 16.0, 64)
    ph = rng.uniform(0.0, 2.0 * np.pi, 64)
    img = np.full((height, width), 128.0)
    for i in range(64):
        kx = 2.0 * np.pi * f[i] * np.cos(th[i])
        ky = 2.0 * np.pi * f[i] * np.sin(th[i])
        img += amp[i] * np.cos(kx * x + ky * y + ph[i])
    white = rng.standard_normal((height, width))
    spec = np.fft.rfft2(white)
    fy = np.fft.fftfreq(height)[:, None]
    fx = np.fft.rfftfreq(width)[None, :]
    mag = np.hypot(fy, fx)
    mag[0, 0] = np.inf
    pink = np.fft.irfft2(spec / mag, s=(height, width))
    pink *= 8.0 / max(pink.std(), 1e-30)
    return np.clip(np.rint(img + pink), 0, 255).astype(np.uint8)


def rectangles_frame(rng: np.random.Generator, height: int, width: int,
                     count: int = 400) -> np.ndarray:
    """Config-3 luma: random axis-aligned rectangles with uniform integer
    intensities in [0, 255] over a uniform random background, uint8."""
    img = np.full((height, width), rng.integers(0, 256), dtype=np.uint8)
    for _ in range(count):
        h = int(rng.integers(8, height // 4))
        w = int(rng.integers(8, width // 4))
        r0 = int(rng.integers(0, height - h))
        c0 = int(rng.integers(0, width - w))
        img[r0:r0 + h, c0:c0 + w] = rng.integers(0, 256)
    return img


def macroblock_losses(rng: np.random.Generator, height: int, width: int, mb: int,
                      fraction: float) -> np.ndarray:
    """(L, 2) top-left corners of lost macroblocks, sorted row-major.

    Only full macroblocks are candidates (a partial bottom strip, e.g. the last
    8 rows of 1080p at mb=16, is never lost), drawn without replacement.
    """
    rows, cols = height // mb, width // mb
    n_mb = rows * cols
    pick = np.sort(rng.choice(n_mb, int(round(fraction * n_mb)), replace=False))
    return np.stack([(pick // cols) * mb, (pick % cols) * mb], axis=1).astype(np.int64)


@dataclass
class FrameCase:
    """A damaged frame plus the per-block area geometry of its lost macroblocks."""

    frame: np.ndarray        # (H, W) uint8 original
    lost: np.ndarray         # (H, W) bool
    corners: np.ndarray      # (L, 2) macroblock top-left corners
    mb: int
    support: int

    @property
    def n_blocks(self) -> int:
        return len(self.corners)

    @property
    def area(self) -> int:
        return self.mb + 2 * self.support

    def damaged(self) -> np.ndarray:
        out = self.frame.astype(np.float64)
        out[self.lost] = 0.0
        return out


def frame_case(workload: Workload) -> FrameCase:
    assert workload.frame is not None
    rng = np.random.default_rng([workload.cid, FRAME_SEED])
    h, w = workload.frame
    if workload.cid == 3:
        frame = rectangles_frame(rng, h, w)
    else:
        frame = texture_frame(rng, h, w)
    corners = macroblock_losses(rng, h, w, workload.macroblock, workload.loss_fraction)
    lost = np.zeros((h, w), dtype=bool)
    mb = workload.macroblock
    for r0, c0 in corners:
        lost[r0:r0 + mb, c0:c0 + mb] = True
    return FrameCase(frame=frame, lost=lost, corners=corners, mb=mb, support=workload.support)


def frame_areas(image: np.ndarray, lost: np.ndarray, corners: np.ndarray, mb: int,
                support: int):
    """Fixed-size areas around each lost macroblock.

    Returns (signals (L, A, A) float64, masks (L, A, A) bool) with A = mb + 2*support.
    Out-of-frame samples carry signal 0 and count as unavailable (mask True);
    every lost pixel of the frame inside the area is masked too
    (BASELINE config 2/3: "lost and unavailable samples set to zero").
    """
    img = np.asarray(image, dtype=np.float64)
    h, w = img.shape
    a = mb + 2 * support
    pad_img = np.zeros((h + 2 * support + mb, w + 2 * support + mb), dtype=np.float64)
    pad_mask = np.ones(pad_img.shape, dtype=bool)
    pad_img[support:support + h, support:support + w] = img
    pad_mask[support:support + h, support:support + w] = lost
    n = len(corners)
    signals = np.empty((n, a, a), dtype=np.float64)
    masks = np.empty((n, a, a), dtype=bool)
    for i, (r0, c0) in enumerate(corners):
        signals[i] = pad_img[r0:r0 + a, c0:c0 + a]
        masks[i] = pad_mask[r0:r0 + a, c0:c0 + a]
    signals[masks] = 0.0
    return signals, masks
