"""B200-native BFV-RNS hot path for LoLa encrypted inference (arXiv 1812.10659).

Device code: paper_1812_10659_b200/csrc (sm_100a CUDA + C++ host), exported
through the C-ABI in include/lola_b200.h and bound here with ctypes.
"""
