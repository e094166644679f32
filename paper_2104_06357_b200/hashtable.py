"""Open-addressing hash accumulator of the hash execution strategy
(reference: /root/reference/pkg/src/semidist/hashtable.py), device-backed.

The table lives in HBM (int64 keys, float64 values, ``capacity`` slots, empty
slots = ``EMPTY_SLOT``); ``build`` inserts in the given order by linear
probing from ``mix32(key) % capacity`` (sd_hash_build, one device thread, so
the slot layout is exactly the reference's) and ``probe_many`` looks keys up
one device thread each (sd_hash_probe).  The engine's shared-memory tables
(csrc/engine.cu) use the same hash and probe sequence.
"""

import numpy as np

from . import _lib

EMPTY_SLOT = np.iinfo(np.int64).max   # hashtable.py:12


def _dev(device=None):
    import torch
    return torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())


def mix32(keys, *, device=None):
    """32-bit avalanche mix of the low 32 bits of each key, as uint64 (hashtable.py:21-29)."""
    import torch
    arr = np.asarray(keys)
    flat = np.ascontiguousarray(arr, dtype=np.int64).reshape(-1)
    dev = _dev(device)
    k = torch.from_numpy(flat).to(dev)
    out = torch.empty(flat.size, dtype=torch.int64, device=dev)
    if flat.size:
        _lib.call(dev, "sd_mix32", k.data_ptr(), flat.size, out.data_ptr(), _lib.stream_handle(dev))
    return out.cpu().numpy().view(np.uint64).reshape(arr.shape)


class HashAccumulator:
    """Fixed-capacity map from column id to float value (hashtable.py:32-106)."""

    def __init__(self, capacity, *, device=None):
        import torch
        capacity = int(capacity)
        if capacity < 1:
            raise ValueError("capacity must be at least 1")
        self.capacity = capacity
        self.device = _dev(device)
        self._tk = torch.full((capacity,), EMPTY_SLOT, dtype=torch.int64, device=self.device)
        self._tv = torch.zeros(capacity, dtype=torch.float64, device=self.device)
        self.size = 0

    @property
    def _keys(self):
        return self._tk.cpu().numpy()

    @property
    def _values(self):
        return self._tv.cpu().numpy()

    def build(self, cols, vals):
        """Reset the table and insert unique keys ``cols`` with ``vals``."""
        import torch
        cols = np.ascontiguousarray(cols, dtype=np.int64).reshape(-1)
        vals = np.ascontiguousarray(vals, dtype=np.float64).reshape(-1)
        if cols.size >= self.capacity:
            raise ValueError(f"{cols.size} entries cannot fit capacity {self.capacity}")
        k = torch.from_numpy(cols).to(self.device)
        v = torch.from_numpy(vals).to(self.device)
        _lib.call(self.device, "sd_hash_build", k.data_ptr() if cols.size else None,
                  v.data_ptr() if cols.size else None, cols.size, self.capacity, self._tk.data_ptr(),
                  self._tv.data_ptr(), _lib.stream_handle(self.device))
        self.size = int(cols.size)

    def probe(self, col):
        """Value stored for ``col``, or ``None`` when absent."""
        values, found = self.probe_many(np.array([col], dtype=np.int64))
        return float(values[0]) if found[0] else None

    def probe_many(self, cols):
        """Vectorized lookup: (values, found) with 0.0 for absent keys."""
        import torch
        cols = np.ascontiguousarray(cols, dtype=np.int64).reshape(-1)
        n = cols.size
        if n == 0 or self.size == 0:
            return np.zeros(n, dtype=np.float64), np.zeros(n, dtype=bool)
        q = torch.from_numpy(cols).to(self.device)
        ov = torch.empty(n, dtype=torch.float64, device=self.device)
        of = torch.empty(n, dtype=torch.uint8, device=self.device)
        _lib.call(self.device, "sd_hash_probe", self._tk.data_ptr(), self._tv.data_ptr(), self.capacity,
                  q.data_ptr(), n, ov.data_ptr(), of.data_ptr(), _lib.stream_handle(self.device))
        return ov.cpu().numpy(), of.cpu().numpy().astype(bool)
