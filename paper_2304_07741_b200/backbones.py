"""Backbones of the BASELINE.json workloads.

PAPER.md:446-447 replaces "all standard convolutions" of its workloads; a
standard conv here is ``groups == 1`` with C_in | C_out or C_out | C_in
(``module.conv_is_target``).  torchvision has ResNet-18, MobileNetV2,
EfficientNet-B0 and VGG-16; the CIFAR ResNet-29 / ResNeXt-29 (2x64d) of
config 3 are not in torchvision and are defined here (3 stages x 3
bottleneck blocks x 3 convs + stem + classifier = 29 layers; ResNeXt-29 2x64d
uses cardinality 2 and bottleneck width 64 per group, so its grouped 3x3
convs are not standard convs and stay as they are).

``build(name, ir_text)`` returns the network with every target replaced by
``CanvasConv2d`` and (for ResNets) its BatchNorms running as the fused BN
post-pass (post.py); ``SPECS`` gives the input shape and class count.
"""

from __future__ import annotations

import torch
from torch import nn

from .module import conv_is_target, replace

SPECS = {
    "resnet18": {"input": (3, 224, 224), "classes": 1000, "kernel_sizes": (3,), "config": 2},
    "resnet29": {"input": (3, 32, 32), "classes": 10, "kernel_sizes": (1, 3), "config": 3, "batch": 512},
    "resnext29_2x64d": {"input": (3, 32, 32), "classes": 10, "kernel_sizes": (1, 3), "config": 3, "batch": 512},
    "mobilenet_v2": {"input": (3, 224, 224), "classes": 1000, "kernel_sizes": (1, 3), "config": 5},
    "efficientnet_b0": {"input": (3, 224, 224), "classes": 1000, "kernel_sizes": (1, 3, 5), "config": 5},
    "vgg16": {"input": (3, 224, 224), "classes": 1000, "kernel_sizes": (3,), "config": 5},
}


class CifarResNeXt(nn.Module):
    """CIFAR ResNet/ResNeXt-29: 3x3 stem (3 -> 64), stages of 3 bottlenecks with
    outputs 256/512/1024 (strides 1/2/2), global pool, linear classifier.
    ``cardinality`` 1 = ResNet-29, 2 = ResNeXt-29 2x64d."""

    def __init__(self, cardinality: int = 1, base_width: int = 64, num_classes: int = 10):
        from torchvision.models.resnet import Bottleneck

        super().__init__()
        self.conv1 = nn.Conv2d(3, 64, 3, padding=1, bias=False)
        self.bn1 = nn.BatchNorm2d(64)
        self.relu = nn.ReLU(inplace=True)
        self._canvas_stem = True  # post.fuse_backbone: fuse bn1 -> relu
        inplanes = 64
        stages = []
        for planes, stride in ((64, 1), (128, 2), (256, 2)):
            blocks = []
            for b in range(3):
                s = stride if b == 0 else 1
                down = None
                if s != 1 or inplanes != planes * 4:
                    down = nn.Sequential(nn.Conv2d(inplanes, planes * 4, 1, stride=s, bias=False), nn.BatchNorm2d(planes * 4))
                blocks.append(Bottleneck(inplanes, planes, s, down, groups=cardinality, base_width=base_width))
                inplanes = planes * 4
            stages.append(nn.Sequential(*blocks))
        self.layer1, self.layer2, self.layer3 = stages
        self.avgpool = nn.AdaptiveAvgPool2d(1)
        self.fc = nn.Linear(inplanes, num_classes)

    def forward(self, x):
        x = self.relu(self.bn1(self.conv1(x)))
        x = self.layer3(self.layer2(self.layer1(x)))
        return self.fc(torch.flatten(self.avgpool(x), 1))


def backbone(name: str) -> nn.Module:
    """Random-init (seeded by the caller) backbone of one workload."""
    import torchvision.models as tvm

    if name == "resnet18":
        return tvm.resnet18(num_classes=1000)
    if name == "resnet29":
        return CifarResNeXt(cardinality=1)
    if name == "resnext29_2x64d":
        return CifarResNeXt(cardinality=2)
    if name == "mobilenet_v2":
        return tvm.mobilenet_v2(num_classes=1000)
    if name == "efficientnet_b0":
        return tvm.efficientnet_b0(num_classes=1000)
    if name == "vgg16":
        return tvm.vgg16(num_classes=1000)
    raise KeyError(name)


def targets(model: nn.Module, kernel_sizes) -> list:
    """(name, conv) of every replacement target, in module order."""
    return [(n, m) for n, m in model.named_modules() if conv_is_target(m) and m.kernel_size[0] in kernel_sizes]


def build(name: str, ir_text: str, *, g: int = 4, fuse_bn: bool = True, factory=None, seed: int = 0) -> tuple[nn.Module, list]:
    """Backbone ``name`` with all standard convs replaced by ``ir_text``.
    Returns (model, replaced names).  ``factory`` as in ``module.replace``."""
    torch.manual_seed(seed)
    m = backbone(name)
    spec = SPECS[name]
    names = replace(m, ir_text, g=g, kernel_sizes=spec["kernel_sizes"], factory=factory)
    if fuse_bn and factory is None:
        from .dense_conv import accelerate_dense
        from .post import fuse_backbone

        fuse_backbone(m)
        accelerate_dense(m)  # ResNet stem + downsample convs on the tcgen05 templates (3xTF32)
    return m, names
