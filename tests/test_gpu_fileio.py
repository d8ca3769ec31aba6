"""The reference's factor / block file formats (lowrank.cpp:601-655,
born.cpp:156-185) written and read from device memory; the expected bytes
are built with numpy directly from the reference's layout."""
import os
import struct

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_1410_0986_b200 as h
    return h.Context(0)


def ref_factor_bytes(U, V, tol, method, perm):
    m, r = U.shape
    n = V.shape[0]
    b = struct.pack("<qqqdqq", m, n, r, tol, method, len(perm))
    b += np.asarray(perm, dtype="<i8").tobytes()
    b += np.ascontiguousarray(U, dtype="<f8").tobytes()  # row-major
    b += np.ascontiguousarray(V, dtype="<f8").tobytes()
    return b


@pytest.mark.parametrize("m,n,r", [(37, 53, 5), (300, 1000, 31), (4, 3, 0), (2000, 9000, 64)])
def test_factor_save_matches_reference_bytes_and_round_trips(ctx, tmp_path, m, n, r):
    from paper_1410_0986_b200 import lowrank as lr
    rng = np.random.default_rng(m + n + r)
    U, V = rng.standard_normal((m, r)), rng.standard_normal((n, r))
    perm = rng.permutation(m).astype(np.int32)
    f = lr.LowRankFactor.from_tensors(ctx, torch.as_tensor(U), torch.as_tensor(V), tol=1e-7,
                                      method=lr.RECURSIVE)
    path = str(tmp_path / "f.bin")
    lr.save_factor(path, f, perm)
    assert open(path, "rb").read() == ref_factor_bytes(U, V, 1e-7, lr.RECURSIVE, perm)
    g, p2 = lr.load_factor(ctx, path)
    assert (g.rows(), g.cols(), g.rank()) == (m, n, r) and g.tol == 1e-7 and g.method == lr.RECURSIVE
    np.testing.assert_array_equal(p2, perm)
    np.testing.assert_array_equal(g.U.cpu().numpy(), U)
    np.testing.assert_array_equal(g.V.cpu().numpy(), V)


def test_factor_load_errors(ctx, tmp_path):
    from paper_1410_0986_b200 import lowrank as lr
    bad = tmp_path / "bad.bin"
    bad.write_bytes(struct.pack("<qqqdqq", 3, 2, 5, 0.0, 0, 0))  # rank > min(m, n)
    with pytest.raises(Exception, match="corrupt factor file"):
        lr.load_factor(ctx, str(bad))
    short = tmp_path / "short.bin"
    short.write_bytes(ref_factor_bytes(np.ones((4, 2)), np.ones((5, 2)), 0.0, 0, [0, 1, 2, 3])[:-16])
    with pytest.raises(Exception, match="truncated factor file"):
        lr.load_factor(ctx, str(short))
    with pytest.raises(Exception, match="cannot read factor"):
        lr.load_factor(ctx, str(tmp_path / "missing.bin"))


def test_block_save_load(ctx, tmp_path):
    from paper_1410_0986_b200 import born
    rng = np.random.default_rng(3)
    B = rng.standard_normal((60, 2049))
    dev = torch.as_tensor(B).cuda()
    path = str(tmp_path / "b.bin")
    born.save_block(ctx, path, dev)
    want = struct.pack("<dd", 60.0, 2049.0) + np.ascontiguousarray(B, dtype="<f8").tobytes()
    assert open(path, "rb").read() == want
    back = born.load_block(ctx, path)
    np.testing.assert_array_equal(back.cpu().numpy(), B)
    # a strided (sub-)block is written as its logical rows
    born.save_block(ctx, path, dev[:, :100])
    np.testing.assert_array_equal(born.load_block(ctx, path).cpu().numpy(), B[:, :100])
    bad = tmp_path / "bad.bin"
    bad.write_bytes(struct.pack("<dd", -1.0, 2.0))
    with pytest.raises(Exception, match="corrupt block file"):
        born.load_block(ctx, str(bad))


def test_block_load_rejects_a_file_larger_than_the_buffer(ctx, tmp_path):
    """hydot_block_load takes the buffer's row capacity: a header larger than
    rows_cap x ld is refused before any device write."""
    import ctypes as C
    import os
    from paper_1410_0986_b200 import born
    from paper_1410_0986_b200._lib import check, lib
    from paper_1410_0986_b200.core import dptr
    B = np.arange(12.0 * 7).reshape(12, 7)
    path = str(tmp_path / "big.bin")
    born.save_block(ctx, path, torch.as_tensor(B).cuda())
    guard = torch.full((5 * 7 + 64,), -1.0, dtype=torch.float64, device="cuda")
    r, c = C.c_int64(), C.c_int64()
    with pytest.raises(ValueError, match="more rows than the buffer"):
        check(lib().hydot_block_load(ctx.h, os.fsencode(path), dptr(guard), 7, 5, C.byref(r), C.byref(c)),
              ctx.h)
    assert bool(torch.all(guard == -1.0))  # nothing written
    with pytest.raises(ValueError, match="leading dimension"):
        check(lib().hydot_block_load(ctx.h, os.fsencode(path), dptr(guard), 6, 12, C.byref(r), C.byref(c)),
              ctx.h)
