"""Decode-time execution of chained SparseGemv layers on one device.

``GemvChain`` runs a sequence of device layers where each product's output
feeds the next product's input (the batch-1 decode pattern), replayed as one
CUDA graph.  Every launch carries the programmatic-dependent-launch attribute,
so inside the graph each GEMV issues its weight loads while its predecessor is
still finishing and only waits (griddepcontrol.wait) before reading x.
"""
from __future__ import annotations

import torch

from .packed import DeviceMatrix


class GemvChain:
    def __init__(self, layers: list[DeviceMatrix], stream: torch.cuda.Stream | None = None):
        if not layers:
            raise ValueError("GemvChain: no layers")
        for a, b in zip(layers, layers[1:]):
            if a.rows != b.cols:
                raise ValueError(f"GemvChain: {a.rows} outputs cannot feed {b.cols} inputs")
        self.layers = layers
        self.stream = stream or torch.cuda.Stream()
        width = max(max(d.rows for d in layers), layers[0].cols)
        self.x = torch.zeros(layers[0].cols, dtype=torch.float32, device="cuda")
        self._bufs = [torch.empty(width, dtype=torch.float32, device="cuda") for _ in range(2)]
        self.graph: torch.cuda.CUDAGraph | None = None
        self.out = None

    @property
    def algorithmic_bytes(self) -> int:
        """Weight-side bytes + x + y of every product."""
        return sum(d.algorithmic_bytes + 4 * d.cols + 4 * d.rows for d in self.layers)

    def _launch_all(self):
        x = self.x
        for i, d in enumerate(self.layers):
            y = self._bufs[i % 2][: d.rows]
            d.spmv_into(x, y, self.stream)
            x = y
        self.out = x

    def run_eager(self):
        with torch.cuda.stream(self.stream):
            self._launch_all()
        return self.out

    def capture(self):
        """Capture one pass as a CUDA graph (workspaces are allocated by a
        warm-up pass first: nothing allocates inside the capture)."""
        self.run_eager()
        self.stream.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(self.stream):
            with torch.cuda.graph(g, stream=self.stream):
                self._launch_all()
        self.graph = g
        return g

    def replay(self):
        if self.graph is None:
            self.capture()
        with torch.cuda.stream(self.stream):
            self.graph.replay()
        return self.out

    def step_host(self, x_host: torch.Tensor, y_host: torch.Tensor):
        """End to end from (pinned) host memory: H2D x, one graph replay, D2H y."""
        with torch.cuda.stream(self.stream):
            self.x.copy_(x_host, non_blocking=True)
            self.graph.replay()
            y_host.copy_(self.out, non_blocking=True)
        self.stream.synchronize()
        return y_host
