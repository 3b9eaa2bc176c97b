"""Per-element order fields and device-resident nodal storage.

Mirrors /root/reference/pkg/src/taudg/fields.py:22-162 for three directions
and nv unknowns per node.  Elements with equal signature (N1, N2, N3) form a
bucket; buckets are ordered ascending by signature and elements ascending by
id inside a bucket (fields.py:34-43).  A NodalField owns ONE flat float64
CUDA tensor; element slot s occupies [node_off[s]*nv, node_off[s+1]*nv) as a
[nv][N3+1][N2+1][N1+1] block (xi fastest) — the layout every kernel reads.
``blocks`` exposes per-bucket views shaped (B, nv, N3+1, N2+1, N1+1).
"""

from __future__ import annotations

import itertools

import numpy as np

_version_counter = itertools.count(1)


class OrderField:
    """Immutable per-element (N1, N2, N3) orders with bucketed layout."""

    def __init__(self, orders):
        orders = np.asarray(orders, dtype=np.int64)
        if orders.ndim != 2 or orders.shape[1] not in (2, 3):
            raise ValueError("orders must have shape (num_elements, 3)")
        if orders.shape[1] == 2:
            orders = np.concatenate([orders, np.zeros((len(orders), 1), np.int64)], axis=1)
        if orders.size and orders.min() < 0:
            raise ValueError("polynomial orders must be >= 0")
        self.orders = orders.copy()
        self.orders.setflags(write=False)
        self.version = next(_version_counter)
        sigs = sorted({tuple(int(v) for v in row) for row in orders})
        self.group_orders = sigs
        self.group_elements = []
        self.element_slot = np.zeros((len(orders), 2), dtype=np.int64)
        for g, sig in enumerate(sigs):
            ids = np.flatnonzero(np.all(orders == np.array(sig), axis=1))
            self.group_elements.append(ids)
            self.element_slot[ids, 0] = g
            self.element_slot[ids, 1] = np.arange(len(ids))
        # slot-order tables
        self.slot_elem = (np.concatenate(self.group_elements) if sigs else np.zeros(0, np.int64))
        self.slot_of_elem = np.empty(len(orders), dtype=np.int64)
        self.slot_of_elem[self.slot_elem] = np.arange(len(orders))
        so = self.orders[self.slot_elem]
        self.slot_orders = so
        self.slot_nodes = np.prod(so + 1, axis=1)
        self.node_off = np.concatenate([[0], np.cumsum(self.slot_nodes)]).astype(np.int64)
        self.group_slot0 = []
        s = 0
        for ids in self.group_elements:
            self.group_slot0.append(s)
            s += len(ids)

    @classmethod
    def uniform(cls, num_elements, n1, n2=None, n3=None):
        n2 = n1 if n2 is None else n2
        n3 = n1 if n3 is None else n3
        return cls(np.tile([n1, n2, n3], (num_elements, 1)))

    @property
    def num_elements(self):
        return len(self.orders)

    @property
    def num_nodes(self):
        return int(self.node_off[-1])

    def dofs(self):
        return self.num_nodes

    def max_order(self):
        return int(self.orders.max())

    def max_order_dir(self, direction):
        return int(self.orders[:, direction - 1].max())

    def same_orders(self, other):
        return self.orders.shape == other.orders.shape and bool(np.all(self.orders == other.orders))

    def __eq__(self, other):
        return self is other

    def __hash__(self):
        return id(self)


class NodalField:
    """Nodal data over all elements, one flat CUDA float64 tensor."""

    __slots__ = ("field", "data", "nv")

    def __init__(self, field: OrderField, data, nv: int):
        self.field = field
        self.data = data
        self.nv = nv

    @classmethod
    def zeros(cls, field: OrderField, nv: int = 1, device="cuda"):
        import torch

        return cls(field, torch.zeros(field.num_nodes * nv, dtype=torch.float64, device=device), nv)

    @classmethod
    def from_slot_array(cls, field, arr, nv, device="cuda"):
        import torch

        t = torch.as_tensor(np.ascontiguousarray(arr, dtype=np.float64)).to(device)
        return cls(field, t.reshape(-1), nv)

    def copy(self):
        return NodalField(self.field, self.data.clone(), self.nv)

    def _check(self, other):
        if other.field is not self.field:
            raise ValueError(f"field mismatch: version {self.field.version} vs {other.field.version}")

    @property
    def blocks(self):
        f = self.field
        out = []
        for g, (sig, ids) in enumerate(zip(f.group_orders, f.group_elements)):
            s0 = f.group_slot0[g]
            n = int(np.prod(np.array(sig) + 1))
            a = int(f.node_off[s0]) * self.nv
            b = a + len(ids) * n * self.nv
            out.append(self.data[a:b].view(len(ids), self.nv, sig[2] + 1, sig[1] + 1, sig[0] + 1))
        return out

    def element(self, e):
        f = self.field
        s = int(f.slot_of_elem[e])
        n1, n2, n3 = (int(v) for v in f.orders[e])
        a = int(f.node_off[s]) * self.nv
        return self.data[a: a + int(f.slot_nodes[s]) * self.nv].view(self.nv, n3 + 1, n2 + 1, n1 + 1)

    def set_element(self, e, values):
        self.element(e).copy_(values)

    def __add__(self, other):
        self._check(other)
        return NodalField(self.field, self.data + other.data, self.nv)

    def __sub__(self, other):
        self._check(other)
        return NodalField(self.field, self.data - other.data, self.nv)

    def __mul__(self, s):
        return NodalField(self.field, self.data * s, self.nv)

    __rmul__ = __mul__

    def add_scaled(self, other, scale):
        self._check(other)
        self.data.add_(other.data, alpha=scale)

    def scale_add(self, scale, other):
        self._check(other)
        self.data.mul_(scale).add_(other.data)

    def norm_inf(self) -> float:
        return float(self.data.abs().max().item()) if self.data.numel() else 0.0

    def all_finite(self) -> bool:
        import torch

        return bool(torch.isfinite(self.data).all().item())

    # --- layout conversion (tests / host I/O) ---------------------------------
    def to_numpy_slots(self):
        return self.data.detach().cpu().numpy()

    def to_oracle_blocks(self):
        """Per-bucket numpy blocks in the oracle's (B, nv, n1, n2, n3) layout."""
        return [b.detach().cpu().numpy().transpose(0, 1, 4, 3, 2).copy() for b in self.blocks]

    def load_oracle_blocks(self, blocks):
        for dst, src in zip(self.blocks, blocks):
            import torch

            dst.copy_(torch.as_tensor(np.ascontiguousarray(np.asarray(src).transpose(0, 1, 4, 3, 2))))
        return self
