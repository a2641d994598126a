"""Host logic of the Krylov graph caches: a cached CUDA graph must never be replayed
for a different operator / preconditioner that happens to reuse a freed object's id."""
import gc

from paper_1712_00403_b200 import krylov


class _Op:
    def apply(self, x, y):
        return y


def test_cache_entry_pins_and_matches_its_callables():
    a, p = _Op(), _Op()
    ent = {"refs": krylov._refs(a.apply, p.apply)}
    assert krylov._same_callables(ent, a.apply, p.apply)        # new bound-method objects, same owners
    assert not krylov._same_callables(ent, p.apply, a.apply)    # swapped roles
    b = _Op()
    assert not krylov._same_callables(ent, b.apply, p.apply)    # another operator
    # the entry holds the owners: deleting the caller's references cannot free them
    ida = id(a)
    del a
    gc.collect()
    assert id(ent["refs"][0][0]) == ida


def test_plain_functions_and_lambdas():
    f = lambda x, y: y  # noqa: E731
    g = lambda x, y: y  # noqa: E731
    ent = {"refs": krylov._refs(f, g)}
    assert krylov._same_callables(ent, f, g) and not krylov._same_callables(ent, g, f)
    assert krylov._fid(f) != krylov._fid(g)
