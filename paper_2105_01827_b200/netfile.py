"""Network layer lists in the reference's file format (pkg/src/gala/profiler.py:9-17, 61-88).

    conv <u_w> <u_h> <c_i> <k_w> <k_h> <c_o>
    fc <n_i> <n_o>
    nonlinear <label>

``parse_network`` / ``load_network`` have the reference's names, semantics and errors
(NetworkParseError with the 1-based line number).  ``network_layers`` turns a parsed list into the
config-5 driver's layers (``resnet.LayerSpec``): the format has no strides, so a convolution followed
by ``nonlinear subsample <s>`` is the stride-s layer (computed at stride 1 and read at every s-th
position -- SURVEY.md 7.3-6), and fc layers keep the reference's padding rule
(``profiler._fc_padded``, profiler.py:117-122).  The network profiler itself (per-layer cost
reports) is out of scope.
"""
from __future__ import annotations

import os
from dataclasses import dataclass

from .errors import NetworkParseError, ParameterError

NETWORKS = os.path.join(os.path.dirname(os.path.abspath(__file__)), "networks")


@dataclass(frozen=True)
class NetLayer:
    """One line of a network file (the reference's profiler.LayerSpec fields)."""

    kind: str                 # "conv" | "fc" | "nonlinear"
    u_w: int | None = None
    u_h: int | None = None
    c_i: int | None = None
    k_w: int | None = None
    k_h: int | None = None
    c_o: int | None = None
    n_i: int | None = None
    n_o: int | None = None
    label: str = ""

    @property
    def is_linear(self) -> bool:
        return self.kind in ("conv", "fc")


def parse_network(text: str) -> list[NetLayer]:
    """Parse the layer-list format; '#' starts a comment; errors carry the line number."""
    out = []
    for line_no, raw in enumerate(text.splitlines(), start=1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        kind, *args = line.split()
        try:
            if kind == "conv":
                if len(args) != 6:
                    raise ValueError(f"conv takes 6 fields, got {len(args)}")
                u_w, u_h, c_i, k_w, k_h, c_o = (int(a) for a in args)
                if min(u_w, u_h, c_i, k_w, k_h, c_o) < 1:
                    raise ValueError("conv dimensions must be positive")
                out.append(NetLayer("conv", u_w=u_w, u_h=u_h, c_i=c_i, k_w=k_w, k_h=k_h, c_o=c_o))
            elif kind == "fc":
                if len(args) != 2:
                    raise ValueError(f"fc takes 2 fields, got {len(args)}")
                n_i, n_o = (int(a) for a in args)
                if min(n_i, n_o) < 1:
                    raise ValueError("fc dimensions must be positive")
                out.append(NetLayer("fc", n_i=n_i, n_o=n_o))
            elif kind == "nonlinear":
                out.append(NetLayer("nonlinear", label=" ".join(args)))
            else:
                raise ValueError(f"unknown layer kind {kind!r}")
        except ValueError as e:
            raise NetworkParseError(line_no, str(e)) from None
    return out


def load_network(name_or_path) -> list[NetLayer]:
    """Read a network file from a path, else from this package's networks/ directory."""
    path = str(name_or_path)
    if not os.path.exists(path):
        path = os.path.join(NETWORKS, path)
    if not os.path.exists(path):
        raise FileNotFoundError(f"network file {name_or_path!r} not found")
    with open(path) as f:
        return parse_network(f.read())


def _next_pow2(x: int) -> int:
    return 1 if x <= 1 else 1 << (x - 1).bit_length()


def fc_padded(n_i: int, n_o: int, n: int) -> tuple[int, int]:
    """(n_i, n_o) after power-of-two padding with n_i raised to >= n_o (profiler.py:117-122)."""
    po = _next_pow2(n_o)
    if po > n:
        raise ParameterError(f"fc output {n_o} exceeds the slot count {n}")
    return max(_next_pow2(n_i), po), po


def _stride_of(label: str) -> int:
    parts = label.split()
    if len(parts) == 2 and parts[0] == "subsample":
        try:
            s = int(parts[1])
        except ValueError:
            raise ParameterError(f"bad subsample label {label!r}") from None
        if s < 1:
            raise ParameterError(f"bad subsample label {label!r}")
        return s
    return 1


def network_layers(specs, names: list[str] | None = None):
    """Linear layers of a parsed network as config-5 driver layers (resnet.LayerSpec).

    A conv followed (before the next linear layer) by ``nonlinear subsample s`` gets stride s;
    square images and kernels only (the driver's frames are square)."""
    from .resnet import LayerSpec

    out, idx = [], [i for i, s in enumerate(specs) if s.is_linear]
    for n, i in enumerate(idx):
        s = specs[i]
        nxt = idx[n + 1] if n + 1 < len(idx) else len(specs)
        stride = 1
        for t in specs[i + 1:nxt]:
            stride *= _stride_of(t.label)
        name = names[n] if names else f"{s.kind}{n}"
        if s.kind == "conv":
            if s.u_w != s.u_h or s.k_w != s.k_h:
                raise ParameterError(f"{name}: the driver runs square images and kernels")
            out.append(LayerSpec(name, "conv", s.c_i, s.c_o, s.k_w, stride, s.u_w))
        else:
            if stride != 1:
                raise ParameterError(f"{name}: fc layers cannot be subsampled")
            out.append(LayerSpec(name, "fc", s.n_i, s.n_o))
    return out
