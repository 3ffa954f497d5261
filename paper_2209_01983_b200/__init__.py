"""paper_2209_01983_b200 -- B200-native SALE hot path (arXiv 2209.01983, ScalSALE).

    from paper_2209_01983_b200 import Sale, configs
    cfg, cycles = configs.config("C4")
    ctx = Sale(cfg)
    ctx.step(cycles)

The compute path is libsale.so (hand-written sm_100a CUDA kernels behind the C
ABI in include/sale.h); this package only marshals arguments.
"""
from . import configs  # noqa: F401


def __getattr__(name):
    if name in ("Sale", "SaleError", "nccl_unique_id", "workspace_bytes"):
        from . import sale
        return getattr(sale, name)
    raise AttributeError(name)
