"""Benchmark matrix registry and cache-backed Matrix Market fetch
(the reference's src/bench/fetch.cpp:16-197 and its
checks in proj/tests/test_bench_cli.cpp:67-147), through `_ellwarp`. CPU
only: the transport is injected, no network; downloads are in-memory ustar
archives gzip-compressed here."""
import gzip
import io
import os
import tarfile

import numpy as np
import pytest

TINY = "%%MatrixMarket matrix coordinate real general\n3 3 4\n1 1 2.0\n2 2 3.0\n3 1 -1.0\n3 3 4.0\n"


@pytest.fixture(scope="module")
def em():
    from paper_1501_00324_b200 import load_ellwarp

    return load_ellwarp()


def tar_of(name, text, *more):
    """ustar archive of (name, text) members."""
    buf = io.BytesIO()
    with tarfile.open(fileobj=buf, mode="w", format=tarfile.USTAR_FORMAT) as t:
        for nm, tx in ((name, text),) + more:
            data = tx.encode()
            info = tarfile.TarInfo(nm)
            info.size = len(data)
            t.addfile(info, io.BytesIO(data))
    return buf.getvalue()


def test_registry(em):
    reg = em.matrix_registry()
    names = [e["alias"] for e in reg]
    assert len(reg) == 15 and len(set(names)) == 15
    assert {"circuit", "qcd", "windtunnel", "heart3k", "heart30k"} <= set(names)
    qcd = next(e for e in reg if e["alias"] == "qcd")
    assert (qcd["group"], qcd["file"], qcd["nrows"]) == ("QCD", "conf5_4-8x8-05", 49152)
    assert all(e["group"] == "" for e in reg if e["alias"].startswith("heart"))


def test_tar_extraction(em):
    tar = tar_of("dir/readme.txt", "x" * 700, ("scircuit/scircuit.mtx", TINY))
    assert em.extract_mtx_from_tar(tar_of("scircuit/scircuit.mtx", TINY)) == TINY.encode()
    assert em.extract_mtx_from_tar(tar) == TINY.encode()  # skips the non-.mtx member
    with pytest.raises(em.FetchError):
        em.extract_mtx_from_tar(tar_of("notes.txt", "hello"))
    with pytest.raises(em.FetchError, match="truncated"):
        em.extract_mtx_from_tar(tar_of("a.mtx", TINY)[:520])


def test_fetch_matrix(em, tmp_path):
    d = str(tmp_path)
    with pytest.raises(em.FetchError) as err:
        em.fetch_matrix("nope", d)
    assert "circuit" in str(err.value) and "qcd" in str(err.value)

    calls = []

    def transport(url):
        calls.append(url)
        return gzip.compress(tar_of("scircuit/scircuit.mtx", "%%MatrixMarket matrix coordinate real general\n"
                                    "170998 170998 1\n1 1 1.0\n"))

    path = em.fetch_matrix("circuit", d, transport=transport)
    assert calls and calls[0].endswith("Hamm/scircuit.tar.gz") and os.path.exists(path)

    def no_network(url):
        raise AssertionError("network touched on a cache hit")

    assert em.fetch_matrix("circuit", d, transport=no_network) == path
    assert em.fetch_matrix("circuit", d, offline=True) == path

    def wrong(url):
        return gzip.compress(tar_of("rma10/rma10.mtx", TINY))

    with pytest.raises(em.FetchError, match="dimension mismatch"):
        em.fetch_matrix("harbor", d, transport=wrong)
    assert not os.path.exists(os.path.join(d, "harbor.mtx"))
    with pytest.raises(em.FetchError, match="uniform_band"):
        em.fetch_matrix("qcd", d, offline=True)
    with pytest.raises(em.FetchError, match="synthetic"):
        em.fetch_matrix("heart3k", d)
    with pytest.raises(em.FetchError, match="no HTTP client"):
        em.fetch_matrix("qcd", d)


def test_load_matrix_spec(em, tmp_path):
    d = str(tmp_path)
    assert em.load_matrix_spec("synthetic:laplacian3d:2,2,2", d).nrows == 8
    qcd = em.load_matrix_spec("qcd", d, offline=True)  # offline: the synthetic stand-in
    lens = np.diff(np.asarray(qcd.row_offsets))
    assert lens.min() == 39 and lens.max() == 39
    assert em.load_matrix_spec("heart3k", d).nrows == 3129


@pytest.mark.gpu
def test_load_matrix_spec_files(em, tmp_path):
    """Paths and cached aliases go through the Matrix Market reader and the
    device CSR build."""
    d = str(tmp_path)
    p = tmp_path / "tiny.mtx"
    p.write_text(TINY)
    m = em.load_matrix_spec(str(p), d)
    assert m.nrows == 3 and list(m.row_offsets) == [0, 1, 2, 4]
    (tmp_path / "harbor.mtx").write_text(TINY)  # a cached alias is read as is, even offline
    assert em.load_matrix_spec("harbor", d, offline=True).nrows == 3
