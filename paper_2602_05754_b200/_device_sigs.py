"""ctypes signatures of libpf_device.so beyond the GEMM entry points (filled as the ABI grows)."""


def register(lib, sig) -> None:  # noqa: D401
    return None
