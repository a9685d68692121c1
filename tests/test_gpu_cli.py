"""CLI compress / decompress through main(argv) on the GPU codec, mirroring
the reference's tests/test_cli.py (file round trips, --preprocess, --stats,
dictionary mismatch errors, the lenient summary, stdin / stdout), checked
against the CPU oracle's stream output."""

import io
import sys
from types import SimpleNamespace

import pytest

import oracle
import synth
from conftest import has_gpu

pytestmark = pytest.mark.gpu

if has_gpu():
    import paper_2404_19391_b200 as z
    from paper_2404_19391_b200.cli import main


@pytest.fixture(scope="module", autouse=True)
def _ready():
    if not has_gpu():
        pytest.skip("no GPU")
    oracle.build()
    synth.build()


def run(argv):
    return main([str(a) for a in argv])


def test_file_roundtrip_matches_oracle(tmp_path, capsys):
    corpus = synth.generate("mixed", 30_000, 12).tobytes()
    src = tmp_path / "in.smi"
    src.write_bytes(corpus)
    comp, back = tmp_path / "c.zs", tmp_path / "b.smi"
    assert run(["compress", "-i", src, "-o", comp, "--preprocess", "--stats"]) == 0
    err = capsys.readouterr().err
    d = z.default_dictionary()
    t = oracle.Tables(d.learned, bytes(sorted(d.identity)))
    want, st = oracle.run_stream(t, corpus, "compress", True, False, 4)
    assert comp.read_bytes() == want
    assert f"lines={st['lines']} in_bytes={len(corpus)} out_bytes={len(want)}" in err
    assert run(["decompress", "-i", comp, "-o", back]) == 0
    want_back, _ = oracle.run_stream(t, want, "decompress", False, False, 4)
    assert back.read_bytes() == want_back


def test_preprocessed_roundtrip(tmp_path):
    """test_cli.py:87-94"""
    src = tmp_path / "in.smi"
    src.write_bytes(b"C3CCCCC3\nc9ccccc9O\n")
    comp, back = tmp_path / "c.zs", tmp_path / "b.smi"
    assert run(["compress", "-i", src, "-o", comp, "--preprocess"]) == 0
    assert run(["decompress", "-i", comp, "-o", back]) == 0
    assert back.read_bytes() == b"C0CCCCC0\nc0ccccc0O\n"


def test_wrong_dictionary_reports_line(tmp_path, capsys):
    """test_cli.py:104-114"""
    src = tmp_path / "one.smi"
    src.write_bytes(b"c1ccccc1\n")
    comp = tmp_path / "c.zs"
    assert run(["compress", "-i", src, "-o", comp]) == 0
    tiny = tmp_path / "tiny.zsd"
    z.save_dictionary(z.Dictionary([b"CC"], "none"), str(tiny))
    assert run(["decompress", "-i", comp, "-o", tmp_path / "x", "-d", tiny]) == 1
    err = capsys.readouterr().err
    assert "line 1" in err and "unknown code" in err


def test_lenient_reports_counts(tmp_path, capsys):
    """test_cli.py:116-123"""
    src = tmp_path / "in.smi"
    src.write_bytes(b"C1CC1\nC5CC\n")
    assert run(["compress", "-i", src, "-o", tmp_path / "c.zs", "--preprocess", "--lenient"]) == 0
    assert "skipped=0 flagged=1" in capsys.readouterr().err


def test_strict_error_exit_code(tmp_path, capsys):
    src = tmp_path / "in.smi"
    src.write_bytes(b"CCO\nC[NH3\nCCO\n")
    assert run(["compress", "-i", src, "-o", tmp_path / "c.zs", "--preprocess"]) == 1
    assert "zsmiles: error: line 2: unclosed '[' at offset 1" in capsys.readouterr().err


def test_dash_stdin_stdout(monkeypatch):
    """test_cli.py:127-140"""
    payload = b"CCO\nCCN\n"
    comp = io.BytesIO()
    monkeypatch.setattr(sys, "stdin", SimpleNamespace(buffer=io.BytesIO(payload)))
    monkeypatch.setattr(sys, "stdout", SimpleNamespace(buffer=comp))
    assert main(["compress", "-i", "-", "-o", "-"]) == 0
    back = io.BytesIO()
    monkeypatch.setattr(sys, "stdin", SimpleNamespace(buffer=io.BytesIO(comp.getvalue())))
    monkeypatch.setattr(sys, "stdout", SimpleNamespace(buffer=back))
    assert main(["decompress"]) == 0
    assert back.getvalue() == payload


def test_missing_input_file(tmp_path, capsys):
    assert run(["compress", "-i", tmp_path / "absent.smi", "-o", tmp_path / "out"]) == 1
    assert "zsmiles: error:" in capsys.readouterr().err
