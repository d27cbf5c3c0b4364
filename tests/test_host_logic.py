"""CPU tier: host-side pieces of the runtime that need no device (reference
tests/test_runtime.py:188-201, 415-456; tests/test_verify.py:210-240)."""

import numpy as np
import pytest

import paper_2507_13204_b200 as krn
from paper_2507_13204_b200 import ExecutionConfig, ShapeMismatch, ViewStorage, load_tensor, save_tensor
from paper_2507_13204_b200.runtime import effective_threads


def vec(name, values):
    return ViewStorage.from_values(name, np.asarray(values, dtype=np.float64))


def test_config_validation(monkeypatch):
    with pytest.raises(ValueError):
        ExecutionConfig(threads=0)
    with pytest.raises(ValueError):
        ExecutionConfig(policy="cpu")
    monkeypatch.setenv("KRN_THREADS", "3")
    assert effective_threads(ExecutionConfig(threads=8)) == 3
    monkeypatch.delenv("KRN_THREADS")
    assert effective_threads(ExecutionConfig(threads=8)) == 8


def test_view_storage_host_semantics():
    a = vec("a", [1.0, 2.0])
    c = a.copy()
    c.buffer[0] = 9.0
    assert a.buffer[0] == 1.0
    assert a.buffer is a.buffer and a.flat.base is a.buffer or a.flat is a.buffer
    z = ViewStorage.zeros("z", (2, 3))
    assert z.extents == (2, 3) and z.size == 6 and z.buffer.tolist() == [[0.0] * 3] * 2
    with pytest.raises(ShapeMismatch):
        ViewStorage(krn.lang.nodes.ViewDescriptor("m", 2), np.zeros(3))
    ro = a.peek()
    with pytest.raises(ValueError):
        ro[0] = 5.0
    assert ViewStorage.from_values("i", [1, 2, 3]).buffer.dtype == np.float64


def test_tensor_round_trips(tmp_path):
    original = vec("t", [1.5, -2.25, 3.125e-7])
    save_tensor(tmp_path / "t.tensor", original)
    loaded = load_tensor(tmp_path / "t.tensor")
    assert loaded.name == "t" and np.array_equal(loaded.buffer, original.buffer)
    m = ViewStorage.from_values("m", np.arange(6, dtype=np.float64).reshape(2, 3))
    save_tensor(tmp_path / "m.tensor", m)
    loaded = load_tensor(tmp_path / "m.tensor", name="renamed")
    assert loaded.name == "renamed" and loaded.extents == (2, 3) and np.array_equal(loaded.buffer, m.buffer)
    values = np.random.default_rng(5).normal(size=32)
    save_tensor(tmp_path / "v.tensor", vec("t", values))
    assert np.array_equal(load_tensor(tmp_path / "v.tensor").buffer, values)


@pytest.mark.parametrize("content", ["f32 1 3\n1.0\n2.0\n3.0\n", "f64 3 2 2 2\n" + "0.0\n" * 8,
                                     "f64 1 3\n1.0\n2.0\n", "nonsense\n"])
def test_malformed_tensor_files(tmp_path, content):
    path = tmp_path / "bad.tensor"
    path.write_text(content)
    with pytest.raises(ShapeMismatch):
        load_tensor(path)


def test_check_gradient_semantics():
    ok = krn.check_gradient([1.0, 2.0], [1.0, 2.0])
    assert ok.passed and ok.max_rel_error == 0.0
    bad = krn.check_gradient([36.0, -36.36, 36.0], [36.0, -36.0, 36.0])
    assert not bad.passed and [e.index for e in bad.failures()] == [(1,)]
    zero_ref = krn.check_gradient([1e-12], [0.0])
    assert zero_ref.passed and zero_ref.max_rel_error == 0.0  # inf rel error is not "finite max"
    with pytest.raises(ShapeMismatch):
        krn.check_gradient([1.0], [1.0, 2.0])


def test_binding_checks_need_no_device():
    lap = krn.load_program("laplacian")
    with pytest.raises(ShapeMismatch, match="missing"):
        krn.execute(lap, "normRes1DLaplacianSQ", {"x": vec("x", [1.0])})
    with pytest.raises(ShapeMismatch, match="unexpected"):
        krn.execute(lap, "normRes1DLaplacianSQ", {"x": vec("x", [1.0]), "b": vec("b", [1.0]), "q": 1.0})
    with pytest.raises(KeyError):
        krn.execute(lap, "nope", {})
    with pytest.raises(ShapeMismatch, match="missing"):
        krn.detect_conflicts(lap, "normRes1DLaplacianSQ", {"x": vec("x", [1.0])})
