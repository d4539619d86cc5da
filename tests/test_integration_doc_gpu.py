"""The ctypes binding shown in INTEGRATION.md (section B) runs as written:
executed against the in-tree library, it decodes reference blobs into
caller-owned arrays and raises the reference's error for a corrupt one."""

import os
import re
import sys
import types

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _binding_module(cuda):
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    code = re.search(r"```python\n(# dcomp/_b200\.py.*?)```", text, re.S).group(1)
    code = code.replace('ctypes.CDLL("libdcomp_b200.so")', "ctypes.CDLL(LIB)")
    # the snippet imports the reference's errors module; point it at ours
    sys.modules.setdefault("dcomp", types.ModuleType("dcomp"))
    sys.modules["dcomp.errors"] = cuda.errors
    mod = types.ModuleType("dcomp_b200_binding")
    mod.LIB = cuda.native.LIB_PATH
    exec(compile(code, "INTEGRATION.md", "exec"), mod.__dict__)
    return mod


def test_integration_snippet_decodes(cuda, oracle):
    mod = _binding_module(cuda)
    rng = np.random.default_rng(4)
    datas = [np.clip(np.round(rng.normal(0, s, n)), -127, 127).astype(np.int8) for s, n in ((5, 3000), (30, 70000), (1, 10))]
    blobs = [oracle.compress_blob(d.view(np.uint8)) for d in datas]
    outs = [np.zeros(d.size, np.int8) for d in datas]
    mod.decode_blobs_into(list(zip(blobs, outs)))
    for d, o in zip(datas, outs):
        assert np.array_equal(d, o)
    bad = bytearray(blobs[1])
    bad[500] ^= 0x20
    with pytest.raises(cuda.CorruptStreamError, match=r"\(chunk 7\)"):
        mod.decode_blobs_into([(blobs[0], np.zeros(3000, np.int8)), (bytes(bad), np.zeros(70000, np.int8))],
                              labels=[3, 7])
