"""Seeded synthetic workloads (input data only; shared by the oracle and the CUDA path)."""
from .gen import (CONFIGS, Workload, image_like, make_csr, plant_duplicate,  # noqa: F401
                  sample_sets, text_like, tiny, uniform_pair)
