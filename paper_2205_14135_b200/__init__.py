"""B200-native (sm_100a) FlashAttention behind the reference ``tatn`` operator surface.

Importing the package does not require a GPU; the compute entry points in
``attention`` require the in-tree ``lib/libtatn_b200.so`` and an sm_100 device.
"""
__all__ = ["attention"]
