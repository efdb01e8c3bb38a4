"""Model descriptions (single-device forward graphs, turned into training graphs).

`mlp`, `alexnet_like` and `vgg16_like` reproduce the reference's toy parity
fixtures node for node (models.py:17-90). `alexnet` and `vgg16` are the real
224x224 ImageNet networks the benchmark configurations name (BASELINE.json
configs 1-3); the reference IR cannot express them (no pooling / LRN /
strided conv), so they use this package's IR extensions:
  * alexnet: torchvision topology, 61,100,840 parameters; conv1 11x11/4 pad 2,
    LRN (size 5, alpha 1e-4, beta 0.75, k 2) after conv1/conv2, 3x3/2 max pools;
  * vgg16: configuration D, 138,357,544 parameters; thirteen 3x3 same convs
    (all reference-expressible) and five 2x2/2 max pools.
No dropout (no reference op; it would add RNG to the parity contract).
"""

from __future__ import annotations

from .ir import Graph, GraphBuilder, OpKind
from .training import TrainingGraphSpec, build_training_graph


def _conv(b: GraphBuilder, name: str, x: str, cin: int, cout: int, k: int = 3, **geom) -> str:
    w = b.variable(f"{name}_w", (k, k, cin, cout))
    bias = b.variable(f"{name}_b", (cout,))
    y = b.add(OpKind.CONV2D, name, (x, w), **geom)
    y = b.add(OpKind.BIAS_ADD, f"{name}_zb", (y, bias))
    return b.add(OpKind.RELU, f"{name}_relu", (y,))


def _fc(b: GraphBuilder, name: str, x: str, nin: int, nout: int, flatten: bool = False,
        relu: bool = True) -> str:
    w = b.variable(f"{name}_w", (nin, nout))
    bias = b.variable(f"{name}_b", (nout,))
    extra = {"flatten_lhs": True} if flatten else {}
    y = b.add(OpKind.MATMUL, name, (x, w), **extra)
    y = b.add(OpKind.BIAS_ADD, f"{name}_zb", (y, bias))
    return b.add(OpKind.RELU, f"{name}_relu", (y,)) if relu else y


def _classifier(b: GraphBuilder, logits: str, batch: int, classes: int, lr: float) -> Graph:
    labels = b.input("labels", (batch, classes))
    loss = b.add(OpKind.SOFTMAX_XENT_LOSS, "loss", (logits, labels))
    fwd = b.build(outputs=(loss,))
    variables = tuple(n.id for n in fwd if n.kind is OpKind.VARIABLE)
    return build_training_graph(TrainingGraphSpec(fwd, loss, lr, variables))


def mlp(batch: int = 64, features: tuple[int, ...] = (32, 16, 10), bias: bool = True,
        lr: float = 0.05, name: str = "mlp") -> Graph:
    b = GraphBuilder(name)
    x = b.input("images", (batch, features[0]))
    layers = len(features) - 1
    for i in range(1, layers + 1):
        w = b.variable(f"fc{i}_w", (features[i - 1], features[i]))
        x = b.add(OpKind.MATMUL, f"fc{i}", (x, w))
        if bias:
            bv = b.variable(f"fc{i}_b", (features[i],))
            x = b.add(OpKind.BIAS_ADD, f"fc{i}_zb", (x, bv))
        if i < layers:
            x = b.add(OpKind.RELU, f"fc{i}_relu", (x,))
    return _classifier(b, x, batch, features[-1], lr)


def alexnet_like(batch: int, lr: float = 0.01) -> Graph:
    b = GraphBuilder("alexnet_like")
    x = b.input("images", (batch, 6, 6, 3))
    x = _conv(b, "conv1", x, 3, 8)
    for i in range(2, 6):
        x = _conv(b, f"conv{i}", x, 8, 8)
    x = _fc(b, "fc6", x, 6 * 6 * 8, 128, flatten=True)
    x = _fc(b, "fc7", x, 128, 128)
    x = _fc(b, "fc8", x, 128, 10, relu=False)
    return _classifier(b, x, batch, 10, lr)


def vgg16_like(batch: int, lr: float = 0.01) -> Graph:
    b = GraphBuilder("vgg16_like")
    x = b.input("images", (batch, 8, 8, 3))
    cin = 3
    for i, cout in enumerate((4, 4, 8, 8, 16, 16, 16, 32, 32, 32, 32, 32, 32), start=1):
        x = _conv(b, f"conv{i}", x, cin, cout)
        cin = cout
    x = _fc(b, "fc14", x, 8 * 8 * 32, 128, flatten=True)
    x = _fc(b, "fc15", x, 128, 128)
    x = _fc(b, "fc16", x, 128, 10, relu=False)
    return _classifier(b, x, batch, 10, lr)


LRN_ATTRS = {"size": 5, "alpha": 1e-4, "beta": 0.75, "bias": 2.0}


def alexnet(batch: int, lr: float = 0.01, lrn: bool = True, image: int = 224,
            classes: int = 1000) -> Graph:
    """AlexNet (torchvision layer shapes) on [batch, 224, 224, 3] NHWC images."""
    b = GraphBuilder("alexnet")
    x = b.input("images", (batch, image, image, 3))
    x = _conv(b, "conv1", x, 3, 64, k=11, stride=4, padding=2)
    if lrn:
        x = b.add(OpKind.LRN, "norm1", (x,), **LRN_ATTRS)
    x = b.add(OpKind.MAX_POOL, "pool1", (x,), window=3, stride=2)
    x = _conv(b, "conv2", x, 64, 192, k=5)
    if lrn:
        x = b.add(OpKind.LRN, "norm2", (x,), **LRN_ATTRS)
    x = b.add(OpKind.MAX_POOL, "pool2", (x,), window=3, stride=2)
    x = _conv(b, "conv3", x, 192, 384)
    x = _conv(b, "conv4", x, 384, 256)
    x = _conv(b, "conv5", x, 256, 256)
    x = b.add(OpKind.MAX_POOL, "pool5", (x,), window=3, stride=2)
    side = ((((image + 4 - 11) // 4 + 1 - 3) // 2 + 1 - 3) // 2 + 1 - 3) // 2 + 1
    x = _fc(b, "fc6", x, side * side * 256, 4096, flatten=True)
    x = _fc(b, "fc7", x, 4096, 4096)
    x = _fc(b, "fc8", x, 4096, classes, relu=False)
    return _classifier(b, x, batch, classes, lr)


VGG16_CONFIG_D = (64, 64, "M", 128, 128, "M", 256, 256, 256, "M", 512, 512, 512, "M",
                  512, 512, 512, "M")


def vgg16(batch: int, lr: float = 0.01, image: int = 224, classes: int = 1000) -> Graph:
    """VGG-16 (configuration D) on [batch, 224, 224, 3] NHWC images."""
    b = GraphBuilder("vgg16")
    x = b.input("images", (batch, image, image, 3))
    cin, side, conv_i, pool_i = 3, image, 0, 0
    for item in VGG16_CONFIG_D:
        if item == "M":
            pool_i += 1
            x = b.add(OpKind.MAX_POOL, f"pool{pool_i}", (x,), window=2, stride=2)
            side //= 2
        else:
            conv_i += 1
            x = _conv(b, f"conv{conv_i}", x, cin, item)
            cin = item
    x = _fc(b, "fc14", x, side * side * cin, 4096, flatten=True)
    x = _fc(b, "fc15", x, 4096, 4096)
    x = _fc(b, "fc16", x, 4096, classes, relu=False)
    return _classifier(b, x, batch, classes, lr)


MODELS = {"mlp": mlp, "alexnet_like": alexnet_like, "vgg16_like": vgg16_like,
          "alexnet": alexnet, "vgg16": vgg16}
