"""B200-native SparCML hot path (arXiv 1802.08021): sparse allreduce of
per-rank (index, value) streams, top-k sparsification and QSGD encoding.

The compute path is ``libsparcml.so`` (C ABI in ``include/sparcml.h``);
``sparcml`` is the thin ctypes binding.  There is no CPU fallback: importing
the binding without the built library raises.
"""
__all__ = ["sparcml", "synth"]
