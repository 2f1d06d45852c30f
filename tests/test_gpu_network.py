"""A network file in the reference's layer-list format (profiler.py:9-17) driven through the config-5
layer objects: every linear layer of a small strided / tiled / padded network decrypts to the plaintext
layer, and one layer's output words equal the CPU oracle's."""
import numpy as np
import pytest

from oracle.plain import conv2d_mod_p, dot_mod_p
from paper_2105_01827_b200.backend import HEParams
from paper_2105_01827_b200.netfile import network_layers, parse_network
from paper_2105_01827_b200.resnet import ConvLayer, FCLayer
from twins import P, Mirror

pytestmark = pytest.mark.gpu

NET = """
# a small ResNet-shaped net: halo-tiled 7x7 stride-2 stem, strided 3x3 and 1x1, c_n = 16 stage, padded fc
conv 70 70 3 7 7 4
nonlinear subsample 2
nonlinear relu
conv 14 14 4 3 3 8
nonlinear subsample 2
conv 28 28 4 1 1 8   # shortcut
nonlinear subsample 2
nonlinear relu
conv 7 7 16 3 3 16
nonlinear avgpool
fc 24 40
"""


def test_parsed_network_runs_layer_by_layer():
    specs = network_layers(parse_network(NET))
    assert [(s.kind, s.stride) for s in specs] == [("conv", 2), ("conv", 2), ("conv", 2), ("conv", 1), ("fc", 1)]
    params = HEParams(n=1024, seed=26)            # frames up to 32 x 32
    rng = np.random.default_rng(6)
    for spec in specs:
        if spec.kind == "fc":
            w = rng.integers(-128, 128, (spec.c_out, spec.c_in)) % P
            x = rng.integers(0, P, spec.c_in)
            fc = FCLayer(spec, w, params)
            masks = fc.layer.draw_masks(3)
            got = fc.shares(fc.forward_device(fc.encrypt_frames(x), masks), masks)
            assert np.array_equal(got, dot_mod_p(w, x, P)), spec.name
            continue
        w = rng.integers(-128, 128, (spec.c_out, spec.c_in, spec.k, spec.k)) % P
        x = rng.integers(0, P, (spec.c_in, spec.size, spec.size))
        layer = ConvLayer(spec, w, params)
        got = layer.decrypt_output(layer.forward_device(layer.encrypt_frames(x)))
        assert np.array_equal(got, conv2d_mod_p(x, w, P)[:, ::spec.stride, ::spec.stride]), spec.name


def test_parsed_network_layer_words_equal_the_oracle():
    from test_gpu_fullsize_words import encrypt_blocks, oracle_kg

    spec = network_layers(parse_network(NET))[1]             # 14x14 -> 16x16 frame, stride 2, c_n = 4
    mir = Mirror(HEParams(n=1024, rns_limbs=3, seed=27))
    rng = np.random.default_rng(7)
    w = rng.integers(-128, 128, (spec.c_out, spec.c_in, spec.k, spec.k)) % P
    x = rng.integers(0, P, (spec.c_in, spec.size, spec.size))
    layer = ConvLayer(spec, w, mir.params)
    mir.sync_keys()
    (oy, ox, fr), = list(layer.frames(x))
    g, c = encrypt_blocks(mir, layer.task, fr)
    out = layer.forward_device([(oy, ox, g)])
    assert np.array_equal(layer.ctx.export_words(out[0][2]), oracle_kg(mir, layer.kg, c))
    assert np.array_equal(layer.decrypt_output(out), conv2d_mod_p(x, w, P)[:, ::2, ::2])
