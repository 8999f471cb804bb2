"""FMNM v2 model container, JSON dumps and CSV traces (io.hpp / io.cpp),
mirroring test_io.cpp, plus cross-checks of the native reader/writer against
the oracle's independent restatement (oracle/fmnm.py) and a committed golden
container (tests/golden/fmnm_v2_small.bin, made by
tests/golden/make_fmnm_golden.py).  Host code only: no GPU needed."""
import json
import os

import numpy as np
import pytest

import fmnm

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "fmnm_v2_small.bin")


@pytest.fixture(scope="module")
def ct():
    import paper_2605_19388_b200.container as c

    return c


def make_dump(ct, seed):
    # test_io.cpp:17-38: layout {2, 3}, independent mode (two models), 4 bins
    import paper_2605_19388_b200 as dfm

    rng = np.random.default_rng(seed)
    layout = dfm.BlockLayout([2, 3])
    models = [dfm.NmfModel(1e-6 + rng.random((2, 4, 3)), 1e-6 + rng.random((2, 3, 6))) for _ in range(2)]
    lam = rng.random((4, 2, 5))
    w = [rng.standard_normal((4, mb, mb)) + 1j * rng.standard_normal((4, mb, mb)) for mb in (2, 3)]
    cfg = ct.ModelConfig(n_sources=2, k_bases=3, iterations=17, seed=seed, sample_rate=8000.0, window_len=256,
                         hop_len=64)
    return ct.ModelDump(cfg, layout, False, models, lam, w)


def test_model_container_round_trip_is_exact(ct, tmp_path):
    # test_io.cpp:47-71
    d = make_dump(ct, 1)
    p = str(tmp_path / "fastmnmf_model.bin")
    ct.save_model(p, d)
    b = ct.load_model(p)
    assert b.layout.sizes == d.layout.sizes and b.shared == d.shared
    assert b.config.k_bases == 3 and b.config.iterations == 17
    assert b.config.sample_rate == 8000.0 and b.config.window_len == 256 and b.config.hop_len == 64
    assert b.config.seed == 1 and b.config.floor == d.config.floor
    assert len(b.models) == 2
    for m0, m1 in zip(d.models, b.models):
        assert np.array_equal(m0.T, m1.T) and np.array_equal(m0.V, m1.V)
    assert np.array_equal(b.lam, d.lam)
    for w0, w1 in zip(d.w, b.w):
        assert np.array_equal(w0, w1)


def test_loader_rejects_foreign_files_and_versions(ct, tmp_path):
    # test_io.cpp:73-87
    p = tmp_path / "fastmnmf_bad.bin"
    p.write_bytes(b"not a model container")
    with pytest.raises(RuntimeError, match="load_model: bad magic"):
        ct.load_model(str(p))
    p.write_bytes(b"FMNM" + (99).to_bytes(4, "little"))
    with pytest.raises(RuntimeError, match="^load_model: unsupported container version$"):
        ct.load_model(str(p))
    with pytest.raises(RuntimeError, match="load_model: cannot open"):
        ct.load_model(str(tmp_path / "missing.bin"))


def test_truncated_container_is_rejected(ct, tmp_path):
    d = make_dump(ct, 3)
    p = tmp_path / "m.bin"
    ct.save_model(str(p), d)
    raw = p.read_bytes()
    p.write_bytes(raw[:-8])
    with pytest.raises(RuntimeError, match="load_model: truncated file"):
        ct.load_model(str(p))


def test_native_writer_matches_oracle_restatement(ct, tmp_path):
    # the native container and the oracle's struct-level restatement of
    # io.cpp:49-82 agree byte for byte, in both directions
    d = make_dump(ct, 5)
    p1, p2 = str(tmp_path / "native.bin"), str(tmp_path / "oracle.bin")
    ct.save_model(p1, d)
    cfg = dict(n_sources=2, k_bases=3, iterations=17, floor=d.config.floor, seed=5, sample_rate=8000.0,
               window_len=256, hop_len=64)
    fmnm.write(p2, cfg, [2, 3], False, [(m.T, m.V) for m in d.models], d.lam, d.w)
    assert open(p1, "rb").read() == open(p2, "rb").read()
    cfg_r, sizes, shared, models, lam, w = fmnm.read(p1)
    assert sizes == [2, 3] and not shared and cfg_r["iterations"] == 17
    assert np.array_equal(lam, d.lam) and all(np.array_equal(a, b) for a, b in zip(w, d.w))


def test_golden_container_loads_bitwise(ct):
    cfg, sizes, shared, models, lam, w = fmnm.read(GOLDEN)
    b = ct.load_model(GOLDEN)
    assert b.layout.sizes == sizes == [2, 3] and b.shared is False and b.config.k_bases == 3
    assert b.config.sample_rate == 8000.0 and b.config.iterations == 17
    for (T, V), m in zip(models, b.models):
        assert np.array_equal(T, m.T) and np.array_equal(V, m.V)
    assert np.array_equal(lam, b.lam)
    for a, c in zip(w, b.w):
        assert np.array_equal(a, c)
    # and the generator still reproduces the committed bytes
    import importlib.util

    spec = importlib.util.spec_from_file_location("mk", os.path.join(os.path.dirname(GOLDEN), "make_fmnm_golden.py"))
    mk = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mk)
    import tempfile

    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "g.bin")
        fmnm.write(p, *mk.instance())
        assert open(p, "rb").read() == open(GOLDEN, "rb").read()


def test_json_debug_dump_carries_the_configuration(ct, tmp_path):
    # test_io.cpp:89-103
    d = make_dump(ct, 2)
    p = tmp_path / "fastmnmf_model.json"
    ct.dump_model_json(str(p), d)
    j = json.loads(p.read_text())
    assert j["config"]["k_bases"] == 3
    assert j["partition"] == [2, 3]
    assert j["share_spectrograms"] is False
    assert len(j["models"]) == 2 and len(j["lambda"]) == 4
    assert j["format_version"] == 2
    assert j["w"][1][0][2][1] == [d.w[1][0][2, 1].real, d.w[1][0][2, 1].imag]


def test_trace_csv_has_one_row_per_recorded_cost(ct, tmp_path):
    # test_io.cpp:105-121
    import paper_2605_19388_b200 as dfm

    rep = dfm.FitReport(np.array([10.0, 8.5, 8.0]), np.array([0.5, 0.25]), 2)
    p = tmp_path / "fastmnmf_trace.csv"
    ct.write_trace_csv(str(p), rep)
    lines = [l for l in p.read_text().splitlines() if l]
    assert lines[0] == "iteration,cost,wall_seconds"
    assert len(lines) == 4
    assert lines[2] == "1,8.5,0.5"


def test_eval_trace_csv_columns(ct, tmp_path):
    # test_io.cpp:141-152
    p = tmp_path / "fastmnmf_eval.csv"
    ct.write_eval_trace_csv(str(p), [(10, 1.5, -100.0, 3.5), (20, 3.0, -120.0, 4.1)])
    lines = p.read_text().splitlines()
    assert lines[0] == "iteration,cumulative_seconds,cost,mean_sdr_improvement"
    assert lines[1].startswith("10,")


def test_dumped_init_round_trips_into_an_init_bundle(ct, tmp_path):
    # the §8(d) protocol: a random_init dumped once as FMNM v2 and loaded back
    # is bitwise the same EM starting point
    import paper_2605_19388_b200 as dfm

    layout = dfm.BlockLayout([4, 4, 4])
    init = dfm.random_init(33, 20, layout, 5, 16, 19388)
    d = ct.ModelDump(ct.ModelConfig(n_sources=5, k_bases=16, iterations=200, seed=19388), layout, True,
                     [init.nmf], init.lambda0, init.w0)
    p = str(tmp_path / "init.bin")
    ct.save_model(p, d)
    back = ct.load_model(p).init_bundle()
    assert np.array_equal(back.nmf.T, init.nmf.T) and np.array_equal(back.nmf.V, init.nmf.V)
    assert np.array_equal(back.lambda0, init.lambda0)
    assert all(np.array_equal(a, b) for a, b in zip(back.w0, init.w0))
