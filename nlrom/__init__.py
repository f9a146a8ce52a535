"""`nlrom` drop-in: the reference package name (pkg/pyproject.toml:6) resolving to the
B200-native implementation in paper_2102_11026_b200."""

import importlib
import sys

_impl = importlib.import_module("paper_2102_11026_b200")
_MODULES = ("mcx", "densenet", "diffops", "elastic", "daereduce", "neucubature", "rdsim", "artifacts",
            "substructure", "posegen", "fullspace", "shard", "cli")


def __getattr__(name):
    if name in _MODULES:
        mod = importlib.import_module(f"paper_2102_11026_b200.{name}")
        sys.modules[f"nlrom.{name}"] = mod
        return mod
    raise AttributeError(name)


class _Finder:
    """Make `import nlrom.<module>` load the implementation module."""

    @staticmethod
    def find_spec(fullname, path=None, target=None):
        if fullname.startswith("nlrom.") and fullname.split(".", 1)[1] in _MODULES:
            import importlib.util
            real = importlib.util.find_spec(f"paper_2102_11026_b200.{fullname.split('.', 1)[1]}")
            spec = importlib.util.spec_from_loader(fullname, _Alias(real.name))
            return spec
        return None


class _Alias:
    def __init__(self, real):
        self.real = real

    def create_module(self, spec):
        return importlib.import_module(self.real)

    def exec_module(self, module):
        pass


sys.meta_path.insert(0, _Finder)
