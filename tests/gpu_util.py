"""TEST INFRASTRUCTURE: zero-copy torch views of raw device pointers returned by the C-ABI."""
import torch

_TYPESTR = {torch.float32: "<f4", torch.bfloat16: "<V2", torch.int32: "<i4", torch.int64: "<i8"}


class _Cai:
    def __init__(self, ptr, n, typestr):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 3}


def device_view(ptr: int, n: int, dtype=torch.float32) -> torch.Tensor:
    if dtype is torch.bfloat16:
        t = torch.as_tensor(_Cai(ptr, n, "<i2"), device="cuda")
        return t.view(torch.bfloat16)
    return torch.as_tensor(_Cai(ptr, n, _TYPESTR[dtype]), device="cuda")


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream
