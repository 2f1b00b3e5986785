"""Device plumbing: CUDA availability, streams, descriptor-table uploads.

PyTorch provides allocation and streams only; all compute is in
libdpm_b200.so.  No CPU fallback exists: without a CUDA device the product
path raises DeviceError.
"""

import numpy as np

from .errors import DeviceError

__all__ = ["require_cuda", "stream_handle", "upload_table"]


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device visible: the B200 score path has no CPU fallback")
    return torch


def stream_handle(stream=None):
    """cudaStream_t of ``stream`` (a torch.cuda.Stream) or torch's current stream."""
    import torch

    s = torch.cuda.current_stream() if stream is None else stream
    return s.cuda_stream


def upload_table(arr, device):
    """Copy a numpy structured array into a device byte tensor."""
    import torch

    raw = np.ascontiguousarray(arr).view(np.uint8).reshape(-1)
    if raw.size == 0:
        raw = np.zeros(16, dtype=np.uint8)
    return torch.from_numpy(raw.copy()).to(device)
