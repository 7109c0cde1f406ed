"""Writers for the reference's model manifest (proj/src/model_io.cpp:93-210:
JSON version 1 + little-endian float32 weight blobs) and IDX byte tensors
(model_io.cpp load_idx), so tests can drive the reference CLI (packnn infer)
with this repo's seeded synthetic networks. Test infrastructure."""
from __future__ import annotations

import json
import struct
from pathlib import Path

import numpy as np


def write_model(net, path: Path) -> Path:
    """A Network (paper_1812_10659_b200.nets) as a manifest: each linear
    stage a conv or dense layer (integer weights, scale 0), a square after
    every stage but the last."""
    path = Path(path)
    c, h, w = net.input_shape
    layers = []
    for k, st in enumerate(net.stages):
        wfile = f"{path.stem}.layer{k}.weights.bin"
        np.asarray(st.weights, dtype="<f4").reshape(-1).tofile(path.parent / wfile)
        if st.is_conv:
            layer = {"kind": "conv", "window": list(st.win), "stride": list(st.stride), "maps": int(st.rows),
                     "inputs": int(st.cols), "weights": wfile, "scale": 0}
            if any(st.pad):
                layer["pad"] = [int(v) for v in st.pad]
        else:
            layer = {"kind": "dense", "outputs": int(st.rows), "inputs": int(st.cols), "weights": wfile, "scale": 0}
        if st.bias is not None:
            bfile = f"{path.stem}.layer{k}.bias.bin"
            np.asarray(st.bias, dtype="<f4").tofile(path.parent / bfile)
            layer["bias"] = bfile
        layers.append(layer)
        if k + 1 < len(net.stages):
            layers.append({"kind": "square"})
    root = {"version": 1, "input": {"channels": c, "height": h, "width": w}, "input_bound": int(net.input_bound),
            "layers": layers}
    path.write_text(json.dumps(root))
    return path


def write_idx(images: np.ndarray, shape, path: Path) -> Path:
    """Records of u8 pixels: magic 0x0000 08 <rank>, big-endian dims."""
    path = Path(path)
    arr = np.asarray(images, dtype=np.uint8).reshape((len(images), *shape))
    with open(path, "wb") as f:
        f.write(bytes([0, 0, 0x08, arr.ndim]))
        for d in arr.shape:
            f.write(struct.pack(">I", d))
        f.write(arr.tobytes())
    return path
