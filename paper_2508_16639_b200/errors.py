"""Error taxonomy of the reference (include/escg/errors.hpp:9-26), mapped from C-ABI return codes."""


class ConfigError(RuntimeError):
    """Invalid runtime configuration (errors.hpp:9-12)."""


class IoError(RuntimeError):
    """Filesystem-level failure (errors.hpp:14-17)."""


class FormatError(RuntimeError):
    """Malformed file content (errors.hpp:19-22)."""


class EngineError(RuntimeError):
    """Simulation aborted: corrupt lattice value, CUDA failure, no device (errors.hpp:24-26)."""


_BY_CODE = {2: ConfigError, 3: IoError, 4: FormatError, 5: EngineError}


def raise_for(code: int, message: str) -> None:
    raise _BY_CODE.get(code, EngineError)(message)
