"""Host <-> device transfers of the public entry point run(): the caller's
float64 unary in, the int8 labels out (ref admm.py:207-252 takes and returns
host numpy arrays).

* Unary upload.  The first time a host buffer is seen it is staged through a
  pinned buffer in 16 MB chunks, the multi-threaded host copy of chunk i+1
  overlapping the DMA of chunk i.  When the same buffer comes back on the
  next call (a serving loop that refills one array) it is page-locked once
  with cudaHostRegister and DMA'd directly from then on: no host copy at all.
  The uploader keeps a reference to that array so its memory cannot be
  reused while registered; a different array unregisters it.  The contents
  are read fresh on every call, so in-place edits between calls are seen.
* Labels download.  The device labels go to a cached pinned buffer, then a
  multi-threaded host copy fills a fresh numpy array the caller owns.
"""
from __future__ import annotations

import numpy as np

CHUNK_BYTES = 16 << 20


def _lib():
    from . import _lib as L
    return L.lib()


class UnaryUploader:
    def __init__(self, n: int, device):
        import torch
        self.n = n
        self.device = device
        self.dev = torch.empty(n, dtype=torch.float64, device=device)
        self._pin = None
        self._done = None            # event after the last staged DMA
        self._last = None            # (ptr, nbytes) of the previous call
        self._registered = None      # (ptr, nbytes, array) page-locked in place
        self.registered_uploads = 0
        self.staged_uploads = 0

    def _unregister(self):
        if self._registered is not None:
            _lib().dope_host_unregister(self._registered[0])
            self._registered = None

    def _register(self, arr: np.ndarray) -> bool:
        if _lib().dope_host_register(arr.ctypes.data, arr.nbytes) != 0:
            return False      # (e.g. already registered by the caller): keep staging
        self._registered = (arr.ctypes.data, arr.nbytes, arr)
        return True

    def upload(self, arr: np.ndarray):
        """float64[n] host array -> self.dev (enqueued on the current stream)."""
        import torch
        if arr.dtype != np.float64 or not arr.flags.c_contiguous or arr.size != self.n:
            arr = np.ascontiguousarray(arr, dtype=np.float64).reshape(-1)
        key = (arr.ctypes.data, arr.nbytes)
        same = self._last == key
        if self._registered is not None and self._registered[:2] != key:
            self._unregister()
        if same and self._registered is None:
            self._register(arr)
        self._last = key
        src = torch.from_numpy(arr)
        if self._registered is not None:
            self.dev.copy_(src, non_blocking=True)
            self.registered_uploads += 1
            return self.dev
        if self._pin is None:
            self._pin = torch.empty(self.n, dtype=torch.float64).pin_memory()
        if self._done is not None:
            self._done.synchronize()      # the previous call's DMA has drained the pinned buffer
        step = max(1, CHUNK_BYTES // 8)
        for s in range(0, self.n, step):
            e = min(self.n, s + step)
            self._pin[s:e].copy_(src[s:e])
            self.dev[s:e].copy_(self._pin[s:e], non_blocking=True)
        self._done = torch.cuda.Event()
        self._done.record(torch.cuda.current_stream(self.device))
        self.staged_uploads += 1
        return self.dev

    def close(self):
        self._unregister()
        self._last = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class LabelDownloader:
    def __init__(self, n: int):
        self.n = n
        self._pin = None

    def fetch(self, labels_dev) -> np.ndarray:
        """uint8/int8[n] device labels -> a fresh int8 numpy array (synchronises)."""
        import torch
        if self._pin is None:
            self._pin = torch.empty(self.n, dtype=torch.int8).pin_memory()
        self._pin.copy_(labels_dev.view(torch.int8), non_blocking=True)
        torch.cuda.current_stream(labels_dev.device).synchronize()
        out = torch.empty(self.n, dtype=torch.int8)
        out.copy_(self._pin)
        return out.numpy()
