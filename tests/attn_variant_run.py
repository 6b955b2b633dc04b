"""Helper for tests/test_gpu_attention_variants.py: one 8B-dims first stage (2 layers) runs a
prefill circuit and a mixed decode circuit; writes the bf16 output activations (raw bytes) to
argv[1]. The attention kernel variants are selected by DS_ATTN_DECODE / DS_ATTN_PROMPT."""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, sys.argv[2])
from paper_2501_14784_b200 import _native as nat  # noqa: E402
from paper_2501_14784_b200 import pipeline as pl  # noqa: E402

dims = pl.MODEL_DIMS["llama3-8b"]
md = pl.model_desc(dims)
st = C.c_void_p()
nat.check(nat.lib.ds_stage_create(0, C.byref(md), 0, 2, 1, 0, pl.WEIGHT_SEED, 1024, 8, C.byref(st)))
page = 256 * 2 * 2 * dims["n_kv_heads"] * dims["d_head"] * 2
nat.check(nat.lib.ds_kv_create(st, page, 1, 24 * page, 0, 0))
out = []
for rows in ([(0, 0, 300, 1, 0, 1), (1, 0, 37, 1, 0, 2), (2, 0, 520, 1, 0, 3)],
             [(0, 300, 1, 1, 1, 1), (1, 37, 1, 1, 1, 2), (2, 520, 90, 1, 0, 3), (3, 0, 1, 1, 1, 4)]):
    arr = (nat.Row * len(rows))(*[nat.Row(slot=r[0], pos=r[1], n_tok=r[2], need_logits=r[3],
                                          is_decode=r[4], reserved=0, req_id=r[5]) for r in rows])
    ids = np.array([11, 22, 33], dtype=np.int32)
    d_ids = C.c_void_p()
    nat.check(nat.lib.ds_dbg_alloc(0, 64, C.byref(d_ids)))
    nat.check(nat.lib.ds_dbg_copy(d_ids, ids.ctypes.data, ids.nbytes))
    nat.check(nat.lib.ds_stage_step(st, 0, arr, len(rows), d_ids if rows[0][4] else None, None))
    nat.check(nat.lib.ds_stage_sync(st))
    ptr, nb, n = C.c_void_p(), C.c_int64(), C.c_int64()
    nat.check(nat.lib.ds_stage_output(st, C.byref(ptr), C.byref(nb), C.byref(n)))
    h = np.zeros(nb.value // 2, dtype=np.uint16)
    nat.check(nat.lib.ds_dbg_copy(h.ctypes.data, ptr, nb.value))
    out.append(h)
nat.lib.ds_stage_destroy(st)
np.concatenate(out).tofile(sys.argv[1])
