"""Layer tables, GPU types and links of the paper's testbed (configuration only).

Inputs of the intra-VW pipeline schedule (PAPER.md
section 4 "Pipelined Model Parallelism Within a VW"). Like the rest
of `workloads/` this module holds data, none of the method's arithmetic: the
partitioner and the pipeline simulator live in oracle/pipeline.py (test
infrastructure) and in the library (paper_2005_14038_b200/csrc/pipeline.cpp).

Models (ResNet-152 and VGG-19 on ImageNet, batch 32):
  * VGG-19 (Simonyan & Zisserman 2014, configuration E): 16 conv3x3 layers with
    bias + fc6/fc7/fc8; 19 weight layers, 143,667,240 params ("548MB").
  * ResNet-152 (He et al. 2016, torchvision v1.5 layout: stride on the 3x3
    conv): stem + 50 bottleneck blocks [3, 8, 36, 3] + fc; 60,192,808 params
    ("230MB"; BN weight/bias counted, running statistics are buffers).
A partition unit is a VGG layer (pooling/ReLU folded into the preceding conv)
or a whole ResNet bottleneck block (a cut inside a residual block would cross
its skip connection; sub-layer partitioning is out of scope).

Per unit: params, forward FLOPs per image (2 x MACs of the convolutions / fc;
BN, ReLU, pooling and the residual add are omitted), output activation
elements per image (what crosses a cut), and resident activation elements per
image (what the unit keeps for its backward pass: every conv output and its
BN/ReLU output; ReLU in place).

GPUs (Table 1): CUDA cores, boost clock, memory. Relative
training speed V=1.00, R=0.76, G=0.72, Q=0.59 is the SURVEY.md 8(d) proxy
(Table 3 Horovod ResNet-152 rates 233/4, 353/8, 415/12 images/s, for V,
R, Q; G from Q scaled by Table 1's cores x boost). Absolute rate: a TITAN V
trains ResNet-152 at 233/4 images/s (Table 3, 4[V] Horovod), i.e. 3 x forward
FLOPs per image (forward + backward = 2 x forward) in 1/58.25 s.

Links: GPUs of a node share PCIe 3.0 x16 (15.75 GB/s);
nodes are connected by 56 Gbps InfiniBand (7 GB/s).

Allocation policies (Table 2): four nodes of four GPUs of
one type each; 4 VWs of 4 GPUs.
"""
from __future__ import annotations

import dataclasses
from typing import Dict, List, Sequence, Tuple

BATCH = 32
FP32 = 4


@dataclasses.dataclass(frozen=True)
class Unit:
    name: str
    params: int
    fwd_flops: int        # per image
    act_out: int          # elements per image leaving the unit (crosses a cut)
    act_resident: int     # elements per image kept until the unit's backward


def vgg19() -> List[Unit]:
    cfg = [64, 64, "M", 128, 128, "M", 256, 256, 256, 256, "M",
           512, 512, 512, 512, "M", 512, 512, 512, 512, "M"]
    units: List[Unit] = []
    c_in, hw = 3, 224
    i = 0
    pending = None
    for j, x in enumerate(cfg):
        if x == "M":
            hw //= 2
            u = pending
            units[-1] = Unit(u.name, u.params, u.fwd_flops, u.act_out // 4, u.act_resident)
            continue
        i += 1
        params = 9 * c_in * x + x
        flops = 2 * 9 * c_in * x * hw * hw
        out = x * hw * hw
        pending = Unit(f"conv{i}", params, flops, out, 2 * out)
        units.append(pending)
        c_in = x
    feat = c_in * hw * hw          # 512 * 7 * 7 = 25088
    for name, n_in, n_out in (("fc6", feat, 4096), ("fc7", 4096, 4096), ("fc8", 4096, 1000)):
        units.append(Unit(name, n_in * n_out + n_out, 2 * n_in * n_out, n_out, 2 * n_out))
    return units


def resnet152() -> List[Unit]:
    units: List[Unit] = []
    # stem: conv 7x7/2 3->64 (no bias) + BN, maxpool 3x3/2 -> 56x56x64
    units.append(Unit("stem", 7 * 7 * 3 * 64 + 2 * 64, 2 * 49 * 3 * 64 * 112 * 112,
                      64 * 56 * 56, 2 * 64 * 112 * 112 + 64 * 56 * 56))
    c_in, hw = 64, 56
    for si, (blocks, width) in enumerate(((3, 64), (8, 128), (36, 256), (3, 512))):
        out_c = 4 * width
        for b in range(blocks):
            stride = 2 if (b == 0 and si > 0) else 1
            hw_out = hw // stride
            params = (c_in * width + 2 * width            # conv1 1x1 + bn1
                      + 9 * width * width + 2 * width     # conv2 3x3 + bn2
                      + width * out_c + 2 * out_c)        # conv3 1x1 + bn3
            flops = (2 * c_in * width * hw * hw + 2 * 9 * width * width * hw_out * hw_out
                     + 2 * width * out_c * hw_out * hw_out)
            resident = 2 * (width * hw * hw + width * hw_out * hw_out + out_c * hw_out * hw_out)
            if b == 0:                                    # downsample 1x1 conv + bn
                params += c_in * out_c + 2 * out_c
                flops += 2 * c_in * out_c * hw_out * hw_out
                resident += 2 * out_c * hw_out * hw_out
            units.append(Unit(f"layer{si + 1}.{b}", params, flops, out_c * hw_out * hw_out,
                              resident))
            c_in, hw = out_c, hw_out
    units.append(Unit("fc", 2048 * 1000 + 1000, 2 * 2048 * 1000, 1000, 2048 + 1000))
    return units


MODELS = {"vgg19": vgg19, "resnet152": resnet152}


@dataclasses.dataclass(frozen=True)
class GPUType:
    name: str
    cores: int
    boost_mhz: int
    mem_gb: float
    speed: float          # relative training speed (SURVEY.md 8(d) proxy)


GPUS: Dict[str, GPUType] = {
    "V": GPUType("TITAN V", 5120, 1455, 12, 1.00),
    "R": GPUType("TITAN RTX", 4608, 1770, 24, 0.76),
    "G": GPUType("GeForce RTX 2060", 1920, 1680, 6, 0.72),
    "Q": GPUType("Quadro P4000", 1792, 1480, 8, 0.59),
}

PCIE_BPS = 15.75e9          # P:14, intra-node
IB_BPS = 56e9 / 8           # P:10, inter-node
# TITAN V training rate: ResNet-152 at 233/4 images/s (Table 3)
V_IMG_PER_S_RESNET152 = 233.0 / 4.0

# Table 2: node of each GPU type; a VW is a list of (type, node)
NODE_OF = {"V": 0, "R": 1, "G": 2, "Q": 3}
POLICIES: Dict[str, Tuple[str, ...]] = {
    "NP": ("VVVV", "RRRR", "GGGG", "QQQQ"),
    "ED": ("VRGQ", "VRGQ", "VRGQ", "VRGQ"),
    "HD": ("VVQQ", "VVQQ", "RRGG", "RRGG"),
}


def v_flops_per_s() -> float:
    """Effective training FLOP/s of a TITAN V (forward + backward = 3 x fwd)."""
    f = sum(u.fwd_flops for u in resnet152())
    return 3.0 * f * V_IMG_PER_S_RESNET152


def vw_gpus(policy: str, vw: int) -> List[Tuple[str, int]]:
    return [(t, NODE_OF[t]) for t in POLICIES[policy][vw]]


def layer_rr_bounds(units: Sequence[Unit], G: int, align: int = 32) -> List[int]:
    """PS shard boundaries of the paper's default placement ("we
    place layers of the model in round-robin fashion over all the parameter
    servers"): unit i goes to shard i mod G. With the parameters stored shard
    by shard (a permutation of the model's order) every shard is one
    contiguous range; inner boundaries are rounded to `align` floats."""
    sizes = [0] * G
    for i, u in enumerate(units):
        sizes[i % G] += u.params
    P = sum(sizes)
    b, acc = [0], 0
    for q in range(G - 1):
        acc += sizes[q]
        x = max(b[-1] + align, int(round(acc / align)) * align)
        b.append(x)
    b.append(P)
    assert all(x < y for x, y in zip(b, b[1:]))
    return b
