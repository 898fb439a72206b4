"""B200-native engine for the iQCC Hamiltonian-dressing hot path (arXiv 2603.08883).

``paper_2603_08883_b200.iqcc`` mirrors the reference's ``namespace iqcc`` API
(PauliSum, dress_single, dress_sequence, compress, expect_sum,
qmf_energy_gradient, gradient, dis_candidates, ...) on top of the C-ABI
engine ``libiqcc_b200.so`` (include/iqcc_b200.h).  Importing ``iqcc`` loads
the CUDA engine and raises ImportError when it is missing; there is no CPU
fallback.
"""
__all__ = ["iqcc", "native"]
