"""B200-native ARCHES uplink channel-estimation hot path.

Hand-written sm_100a kernels behind a C ABI (`include/arches.h`,
`lib/libarches.so`), driven from Python through ctypes:

  engine.ArchesPlan / engine.SlotEngine   batched device pipeline (performance path)
  compat                                   drop-in replacements with the reference signatures

Reference: /root/reference/pkg/src/ranswitch (pure Python simulator).
"""
__version__ = "0.1.0"
