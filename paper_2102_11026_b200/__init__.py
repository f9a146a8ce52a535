"""B200-native DAE-subspace Newton-step hot path of arXiv 2102.11026 (reference package `nlrom`).

Modules mirror the reference API (SPEC.md modules): mcx, densenet, diffops, elastic,
daereduce, neucubature, rdsim. The hot path runs in libnlrom_b200.so (sm_100a CUDA,
C ABI in include/nlrom_b200.h); `import nlrom` resolves to this package.
"""

__version__ = "0.1.0"

from . import mcx  # noqa: F401  (pure value type, no device needed)


def __getattr__(name):
    import importlib
    if name in ("densenet", "diffops", "elastic", "daereduce", "neucubature", "rdsim", "session", "synth",
                "problem", "_lib", "posegen", "fullspace", "artifacts", "substructure", "shard", "cli"):
        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
