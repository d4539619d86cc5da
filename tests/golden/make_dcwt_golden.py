"""Golden DCWT files written by the REFERENCE's dcwt module (run here, where
/root/reference is importable; the outputs are committed):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_dcwt_golden.py
"""
import os

import numpy as np
from dcomp import ActivationStats, WeightTensor, dcwt

HERE = os.path.dirname(os.path.abspath(__file__))
rng = np.random.default_rng(0)
tensors = [WeightTensor("a", rng.normal(0, 1, (4, 6))), WeightTensor("b.weight", rng.normal(0, 1, (1, 1))),
           WeightTensor("longer/name.2", rng.normal(0, 1, (7, 3))), WeightTensor("fc", rng.normal(0, 0.2, (64, 96)))]
dcwt.write_weights(os.path.join(HERE, "ref_f64.dcwt"), tensors)
dcwt.write_weights(os.path.join(HERE, "ref_f32.dcwt"), tensors, dtype=np.float32)
dcwt.write_weights(os.path.join(HERE, "ref_i8.dcwt"), [("q", np.array([[1, -2], [127, -127]], dtype=np.int8))],
                   dtype=np.int8)
dcwt.write_stats(os.path.join(HERE, "ref_stats.json"),
                 [ActivationStats(t.name, np.abs(rng.normal(0, 1, t.values.shape[1])) + 0.01) for t in tensors])
