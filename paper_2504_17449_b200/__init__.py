# SPDX-License-Identifier: Apache-2.0
"""B200-native batched multi-tenant hPLM forward pass (HMI, arXiv 2504.17449)."""
