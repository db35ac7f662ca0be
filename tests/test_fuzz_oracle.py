"""The differential fuzz's determinism claims, checked on the oracle alone (no GPU).

gxin/fuzzprog.py builds programs and batches whose result must not depend on the order the
events run in (observe maps with event-unique keys, write-only
commutative accumulators) nor on the per-thread shard assignment (S4: SUM-folded 64-bit ADDs).
If a generated case broke that, the GPU would have no single correct answer and
tests/test_gpu_fuzz.py could not demand bit-exact parity.  So every case is run through the
oracle in index order, reversed, shuffled, and with 64 per-thread shards (O10 --perm /
--pt-shards), and all compared outputs must agree -- maps, ringbuf multisets, stats and R0
(mapped back to the event index)."""
import numpy as np
import pytest

from oracle.oracle import Oracle
import fuzz_util as fu


def _run(texts, ev, seed, order=None, pt_shards=None):
    env = Oracle()
    if pt_shards:
        env.set_pt_shards(pt_shards)
    fds, prog = fu.setup(env, texts, seed)
    r0 = env.run(ev, prog, order=order)
    return r0, fu.outputs(env, fds)


@pytest.mark.parametrize("block", range(6))
def test_fuzz_cases_are_order_and_shard_invariant(block):
    for seed in range(block * 40, block * 40 + 40):
        texts, ev = fu.case(seed)
        n = len(ev)
        r0, out = _run(texts, ev, seed)
        rng = np.random.default_rng(seed)
        for order, shards in ((np.arange(n)[::-1], None), (rng.permutation(n), None), (None, 64)):
            r0b, outb = _run(texts, ev, seed, order=order, pt_shards=shards)
            bad = np.nonzero(r0 != r0b)[0]
            assert bad.size == 0, (seed, "R0 order-sensitive", bad[:4], texts)
            for k in out:
                assert out[k] == outb[k], (seed, k, fu.first_diff(out[k], outb[k]), texts)


def test_fuzz_cases_exercise_every_path():
    """The grammar reaches what the GPU fuzz must cover: each helper error branch and each
    atomic op/width appears in the generated, accepted programs."""
    import re
    seen = set()
    for seed in range(120):
        texts, _ = fu.case(seed)
        for t in texts:
            seen |= set(re.findall(r"\b(atomic_(?:fetch_)?(?:add|or|and|xor)(?:32|64)|xchg(?:32|64)|cmpxchg(?:32|64)|"
                                   r"ldxs[bhw]|call \d+|mapval|jsgt32|mov64 r4, [0-3])\b", t))
    for op in ("add", "or", "and", "xor"):
        for w in ("32", "64"):
            assert f"atomic_{op}{w}" in seen and f"atomic_fetch_{op}{w}" in seen, (op, w)
    for x in ("xchg32", "xchg64", "cmpxchg32", "cmpxchg64", "ldxsb", "ldxsh", "ldxsw", "call 1", "call 2",
              "call 130", "mapval", "mov64 r4, 0", "mov64 r4, 1", "mov64 r4, 2", "mov64 r4, 3"):
        assert x in seen, x
