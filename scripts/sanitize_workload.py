"""Small workload that launches every kernel of libariann_fss.so once or twice,
for compute-sanitizer (memcheck / racecheck / initcheck / synccheck)."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_04593_b200 import _dev, _lib, dealer, fss, keyfile, nn_ops, prg, runtime, shard  # noqa: E402
from paper_2006_04593_b200.sharing import encode_fixed, share  # noqa: E402

torch.cuda.set_device(0)
rng = np.random.default_rng(1)
for n, N in ((32, 3000), (12, 513), (63, 77)):
    a, k0, k1 = fss.keygen_cmp(n, rng, N)
    x = rng.integers(0, 1 << n, N, dtype=np.uint64)
    fss.eval_cmp(0, k0, x)
    fss.eval_cmp(1, k1, x, return_levels=True)
    a, e0, e1 = fss.keygen_eq(n, rng, N)
    fss.eval_eq(0, e0, x)
    # ARNK tile kernels: TMA path, and the unaligned last tile (odd count) fallback
    fss.unpack_keys(fss.deserialize_keys(fss.serialize_keys(fss.pack_keys(k0, k1))))
    fss.unpack_keys(fss.deserialize_keys(fss.serialize_keys(fss.pack_keys(e0, e1))))
    q0, q1 = k0.take(slice(0, N - 2)), k1.take(slice(0, N - 2))
    fss.unpack_keys(fss.deserialize_keys(fss.serialize_keys(fss.pack_keys(q0, q1))))
fss.keygen_eq(64, rng, 100)
# ARNK pack through TMA tensor maps (level stride a multiple of 16): whole
# batches, ragged prefixes (zero-filled box elements), 16-aligned views
for n, N in ((32, 3008), (12, 512), (63, 64)):
    a, k0, k1 = fss.keygen_cmp(n, rng, N)
    a, e0, e1 = fss.keygen_eq(n, rng, N)
    for lo, hi in ((0, N), (0, N - 5), (16, N - 3)):
        fss._pack_device(k0.take(slice(lo, hi)))
        fss._pack_device(e0.take(slice(lo, hi)))
# sharded dealer (tape slices) and streaming key files
for r in range(3):
    shard.keygen_cmp_shard(32, np.random.default_rng(4), 1001, r, 3)
    shard.keygen_eq_shard(40, np.random.default_rng(4), 1001, r, 3)
a, k0, k1 = fss.keygen_cmp(32, rng, 999)
keyfile.save_keys("/tmp/sanitize_keys.arnk", k0, k1, chunk=100)
keyfile.load_keys("/tmp/sanitize_keys.arnk", chunk=64)
keyfile.load_keys("/tmp/sanitize_keys.arnk", party=1, chunk=333)
# evaluation straight from payload rows (record loads up to the payload's end)
for kind, n, N in (("cmp", 32, 999), ("cmp", 12, 77), ("cmp", 63, 33), ("eq", 5, 101), ("eq", 64, 17),
                   ("eq", 32, 64)):
    kg = fss.keygen_cmp if kind == "cmp" else fss.keygen_eq
    a, k0, k1 = kg(n, rng, N)
    pk = fss.PackedKeyBatch(fss.KIND_CMP if kind == "cmp" else fss.KIND_EQ, 1, n, fss._pack_device(k1))
    (fss.eval_cmp if kind == "cmp" else fss.eval_eq)(1, pk, a)
fss.keygen_cmp(16, rng, 64, out_bits=40)
prg.expand(rng.integers(0, 256, (1000, 16), dtype=np.uint8), 3)
seeds = torch.randint(0, 256, (1024, 16), dtype=torch.uint8, device="cuda")
out = torch.empty((1024, 48), dtype=torch.uint8, device="cuda")
_lib.call("fss_aes_mmo_expand", _dev.ptr(seeds), 1024, 3, _dev.ptr(out),
          ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
prg.mask_stream(bytes(range(16)), 3, 1001, 32)
xs = share(encode_fixed(rng.uniform(-10, 10, (2, 8, 8)), 3, 32), rng, precision=3)
d = dealer.make_dealer(32, seed=2)
runtime.run_local_pair(lambda s: nn_ops.maxpool(s, xs[s.party], 2,
                                                d.for_party(s.party).maxpool(8, 2, 2, planes=2), 2))
runtime.run_local_pair(lambda s: nn_ops.maxpool_k2(s, xs[s.party],
                                                   d.for_party(s.party).maxpool_k2(8, planes=2)))
# host pipeline with a small chunk so several chunks run
fss.PIPELINE_MIN, fss.PIPELINE_CHUNK = 1 << 10, 1 << 9
a, k0, k1 = fss.keygen_cmp(32, rng, 3000)
xh = torch.from_numpy(rng.integers(0, 1 << 32, 3000, dtype=np.uint64).view(np.int64)).pin_memory()
fss.eval_cmp(0, k0, xh.view(torch.uint64))
torch.cuda.synchronize()
print("sanitize workload done")
