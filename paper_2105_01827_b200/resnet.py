"""Config 5: every linear layer of a ResNet-18-shaped network at 224x224x3 (BASELINE.json configs[4]).

The reference executes only stride-1 convolutions of images that fit one
ciphertext (`conv.py:73-82`; strides and larger images are non-goals,
`SPEC.md:15`, `SPEC.md:354`).  Config 5 is built from the same kernel-grouping
primitive with three host-side rules:

* **frame embedding** -- an s x s feature map sits in the top-left of an
  F x F frame, F the next power of two (56->64, 28->32, 14->16, 7->8), so
  c_n = n / F^2 channels pack per ciphertext; the kernel-grouping masks treat
  frame pixels outside the image as zero (verified against conv2d_mod_p,
  SURVEY.md A.2);
* **halo tiling** -- images larger than one frame (conv1 at 224x224) are cut
  into F x F frames overlapping by the kernel radius; each frame's interior
  (F - 2h)^2 outputs are exact;
* **stride as subsampling** -- a stride-2 convolution is the stride-1
  same-padded convolution read at even positions; the parties subsample
  their plaintext shares (free).

The final FC (512 -> 1000) is padded to 1024 x 1024 (`profiler._fc_padded`,
profiler.py:117-122) and runs as a paired GALA dot product.  Every layer takes
a fresh encrypted input (the garbled-circuit non-linear steps between layers
are out of scope).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .backend import HEParams, context
from .conv import ConvTask, KernelGroupingConv, encode_channel_blocks
from .errors import ParameterError
from .matvec import GalaFC


@dataclass(frozen=True)
class LayerSpec:
    name: str
    kind: str            # "conv" | "fc"
    c_in: int
    c_out: int
    k: int = 1
    stride: int = 1
    size: int = 1        # input spatial size (square)

    @property
    def out_size(self) -> int:
        return (self.size + self.stride - 1) // self.stride


def resnet18_224() -> list[LayerSpec]:
    """The 21 linear layers of ResNet-18 (ImageNet, 224x224x3, 1000 classes)."""
    L = [LayerSpec("conv1", "conv", 3, 64, 7, 2, 224)]
    for b in range(2):
        L.append(LayerSpec(f"layer1.{b}.conv1", "conv", 64, 64, 3, 1, 56))
        L.append(LayerSpec(f"layer1.{b}.conv2", "conv", 64, 64, 3, 1, 56))
    c, s = 64, 56
    for stage, co in ((2, 128), (3, 256), (4, 512)):
        L.append(LayerSpec(f"layer{stage}.0.conv1", "conv", c, co, 3, 2, s))
        L.append(LayerSpec(f"layer{stage}.0.conv2", "conv", co, co, 3, 1, s // 2))
        L.append(LayerSpec(f"layer{stage}.0.downsample", "conv", c, co, 1, 2, s))
        L.append(LayerSpec(f"layer{stage}.1.conv1", "conv", co, co, 3, 1, s // 2))
        L.append(LayerSpec(f"layer{stage}.1.conv2", "conv", co, co, 3, 1, s // 2))
        c, s = co, s // 2
    L.append(LayerSpec("fc", "fc", 512, 1000))
    return L


def _next_pow2(x: int) -> int:
    return 1 << max(0, math.ceil(math.log2(x)))


class ConvLayer:
    """One (possibly strided, possibly tiled) convolution on kernel-grouping frames."""

    def __init__(self, spec: LayerSpec, kernels: np.ndarray, params: HEParams, shard_blocks: bool = False):
        """``shard_blocks``: split the layer's physical output ciphertexts across the ranks of the
        process group (`sharding.ShardedKernelGroupingConv`: inputs broadcast from rank 0, outputs
        gathered on rank 0) -- the latency form of config 5 on several GPUs."""
        self.spec, self.params = spec, params
        n = params.n
        h = spec.k // 2
        frame = _next_pow2(spec.size)
        max_frame = int(math.isqrt(n))
        if frame > max_frame:                     # halo tiling
            frame = max_frame
        self.frame, self.halo = frame, h
        self.tiled = spec.size > frame
        self.interior = frame - 2 * h if self.tiled else spec.size
        self.tiles = math.ceil(spec.size / self.interior) if self.tiled else 1
        task = ConvTask(frame, frame, spec.c_in, spec.k, spec.k, spec.c_out, kernels, params)
        if spec.c_in % task.channels_per_ct or spec.c_out % task.channels_per_ct:
            raise ParameterError(f"{spec.name}: channels do not pack into {frame}x{frame} frames")
        self.task = task
        # every kept output pixel reads inside the frame's zero margin (or the tile's halo)
        margin_ok = self.tiled or frame - spec.size >= h
        if shard_blocks:
            from .sharding import ShardedKernelGroupingConv

            self.kg = ShardedKernelGroupingConv(task, band_only=margin_ok)
        else:
            self.kg = KernelGroupingConv(task, band_only=margin_ok)
        self.ctx = self.kg.ctx

    @property
    def plaintext_bytes(self) -> int:
        kg = getattr(self.kg, "local", self.kg)
        return kg.resident_bytes if kg is not None else 0

    def frames(self, x: np.ndarray):
        """Yield (origin_y, origin_x, frame array) covering the input x [c_in][s][s]."""
        s, F, h = self.spec.size, self.frame, self.halo
        if not self.tiled:
            fr = np.zeros((self.spec.c_in, F, F), dtype=np.int64)
            fr[:, :s, :s] = x
            yield 0, 0, fr
            return
        I = self.interior
        for ty in range(self.tiles):
            for tx in range(self.tiles):
                oy, ox = ty * I - h, tx * I - h
                fr = np.zeros((self.spec.c_in, F, F), dtype=np.int64)
                y0, y1 = max(0, oy), min(s, oy + F)
                x0, x1 = max(0, ox), min(s, ox + F)
                fr[:, y0 - oy:y1 - oy, x0 - ox:x1 - ox] = x[:, y0:y1, x0:x1]
                yield oy, ox, fr

    def encrypt_frames(self, x: np.ndarray):
        """Client side: encrypted physical inputs per frame ([n_ib][2][L][N] each)."""
        import torch

        out = []
        for oy, ox, fr in self.frames(x):
            blocks = encode_channel_blocks(self.task, fr)
            cts = torch.stack([self.ctx.encrypt_physical(self.ctx.physical(b.slots)) for b in blocks])
            out.append((oy, ox, cts))
        return out

    def forward_device(self, enc_frames):
        if len(enc_frames) > 1 and self.kg.batchable:   # halo tiles share every launch
            import torch

            outs = self.kg.forward_device_batch(torch.stack([cts for _, _, cts in enc_frames]))
            return [(oy, ox, outs[i]) for i, (oy, ox, _) in enumerate(enc_frames)]
        return [(oy, ox, self.kg.forward_device(cts)) for oy, ox, cts in enc_frames]

    def decrypt_output(self, outs) -> np.ndarray:
        """Decrypt, assemble the stride-1 map and subsample by the stride -> [c_out][out][out]."""
        s, F, h = self.spec.size, self.frame, self.halo
        c_n, n = self.kg.c_n, self.params.n
        full = np.zeros((self.spec.c_out, s, s), dtype=np.int64)
        for oy, ox, cts in outs:
            chans = []
            for ob in range(self.kg.n_ob):
                phys = self.ctx.decrypt_physical(cts[ob // self.kg.pair])
                row = ob % self.kg.pair
                chans.append(phys[row * n:(row + 1) * n].reshape(c_n, F, F))
            fmap = np.concatenate(chans)                       # [c_out][F][F]
            if not self.tiled:
                full[:] = fmap[:, :s, :s]
            else:
                I = self.interior
                y0, x0 = oy + h, ox + h
                y1, x1 = min(s, y0 + I), min(s, x0 + I)
                full[:, y0:y1, x0:x1] = fmap[:, h:h + (y1 - y0), h:h + (x1 - x0)]
        st = self.spec.stride
        return full[:, ::st, ::st]


class FCLayer:
    """512 -> 1000 padded to a power-of-two 1024 x 1024 GALA dot product."""

    def __init__(self, spec: LayerSpec, w: np.ndarray, params: HEParams):
        self.spec, self.params = spec, params
        rows, cols = _next_pow2(spec.c_out), _next_pow2(spec.c_in)
        side = max(rows, cols)
        wp = np.zeros((side, side), dtype=np.int64)
        wp[:spec.c_out, :spec.c_in] = w
        self.side = side
        self.layer = GalaFC(wp, params)
        self.ctx = self.layer.ctx

    @property
    def plaintext_bytes(self) -> int:
        return int(sum(b[1].numel() for b in self.layer.blocks) * 8)

    def encrypt_frames(self, x: np.ndarray):
        xp = np.zeros(self.side, dtype=np.int64)
        xp[:self.spec.c_in] = x
        return self.layer.encrypt_input(xp)

    def forward_device(self, cts, masks):
        return self.layer.forward_device(cts, masks)

    def shares(self, masked, masks) -> np.ndarray:
        full = (self.layer.client_shares(masked) + self.layer.server_shares(masks)) % self.params.p
        return full[:self.spec.c_out]


class ResNet18Linear:
    """All ResNet-18 linear layers with resident encoded weights on one GPU."""

    def __init__(self, params: HEParams | None = None, seed: int = 2105, layers=None, only=None,
                 shard_blocks: bool = False):
        """``only``: indices of the layers this process serves (multi-GPU layer partition,
        `sharding.partition_layers`); the others get weights drawn (same stream) but no GPU state."""
        self.params = params or HEParams(n=4096, rns_limbs=3, seed=5)
        self.specs = layers or resnet18_224()
        rng = np.random.default_rng(seed)
        p = self.params.p
        keep = set(range(len(self.specs))) if only is None else set(only)
        self.weights, self.layers = [], []
        for i, spec in enumerate(self.specs):
            if spec.kind == "fc":
                w = rng.integers(-128, 128, (spec.c_out, spec.c_in)) % p
                self.layers.append(FCLayer(spec, w, self.params) if i in keep else None)
            else:
                w = rng.integers(-128, 128, (spec.c_out, spec.c_in, spec.k, spec.k)) % p
                self.layers.append(ConvLayer(spec, w, self.params, shard_blocks=shard_blocks) if i in keep else None)
            self.weights.append(w)
        self.ctx = context(self.params)

    @property
    def plaintext_bytes(self) -> int:
        return sum(l.plaintext_bytes for l in self.layers if l is not None)

    def random_input(self, i: int, rng) -> np.ndarray:
        spec = self.specs[i]
        p = self.params.p
        if spec.kind == "fc":
            return rng.integers(0, p, spec.c_in)
        return rng.integers(0, p, (spec.c_in, spec.size, spec.size))


def layer_costs(specs, measured: dict | None = None) -> list[float]:
    """Per-layer cost estimates for the multi-GPU layer partition: measured ms per layer name
    where known (e.g. `profiles/r1_resnet18_224.jsonl`), else the plaintext MAC count
    c_in c_out k^2 s^2 / stride^2 scaled to the same unit."""
    measured = measured or {}
    macs = [sp.c_in * sp.c_out * sp.k * sp.k * sp.out_size * sp.out_size for sp in specs]
    known = [(measured[sp.name], m) for sp, m in zip(specs, macs) if sp.name in measured]
    scale = sum(ms for ms, _ in known) / max(1, sum(m for _, m in known)) if known else 1.0
    return [float(measured.get(sp.name, m * scale)) for sp, m in zip(specs, macs)]
