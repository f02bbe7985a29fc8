"""ctypes signatures of libpf_host.so (filled as the ABI grows)."""


def register(lib, sig) -> None:  # noqa: D401
    return None
