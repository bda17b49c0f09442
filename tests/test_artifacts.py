"""Artefact drop-in: rom.npz (cli.py:221-248) and CSV writers (cli.py:39-50)
interoperate with files written by the unmodified reference."""

import numpy as np
import pytest
import scipy.sparse as sp


def _fom(golden_dir):
    from paper_2310_04734_b200 import mor
    z = np.load(golden_dir / "frozen_fom.npz")
    K, M, b, c = sp.csc_matrix(z["K"]), sp.csc_matrix(z["M"]), z["b"], z["c"]
    return mor.FullOrderModel(stiffness=lambda f: K, mass=lambda f: M, load=lambda f: b, c_out=c, n=len(b))


def test_csv_bytes_match_reference_writer(golden_dir, tmp_path):
    from paper_2310_04734_b200 import artifacts
    v = np.load(golden_dir / "frf_ref_values.npz")
    rows = [[f, y.real, y.imag, 20.0 * np.log10(max(abs(y), 1e-300) / 20e-6), int(w)]
            for f, y, w in zip(v["freqs"], v["frf"], v["window_index"])]
    out = tmp_path / "frf_mor.csv"
    artifacts.write_csv(out, ["f_hz", "re_p", "im_p", "abs_db", "window"], rows)
    assert out.read_bytes() == (golden_dir / "frf_ref.csv").read_bytes()


def test_load_reference_rom_container(golden_dir):
    from paper_2310_04734_b200 import artifacts
    roms = artifacts.load_roms(golden_dir / "rom_ref.npz", _fom(golden_dir))
    assert [r.window for r in roms] == [(10.0, 50.0), (50.0, 100.0)]
    assert roms[0].converged and not roms[0].stalled and roms[1].stalled
    assert roms[0].r == 4 and roms[1].r == 2
    assert roms[0].error_log == [(10.0, 1e-3), (50.0, 2e-3)]


def test_rom_container_round_trip(golden_dir, tmp_path):
    from paper_2310_04734_b200 import artifacts
    roms = artifacts.load_roms(golden_dir / "rom_ref.npz", _fom(golden_dir))
    artifacts.save_roms(tmp_path / "rom.npz", roms)
    again = artifacts.load_roms(tmp_path / "rom.npz", _fom(golden_dir))
    ref = np.load(golden_dir / "rom_ref.npz")
    mine = np.load(tmp_path / "rom.npz")
    assert sorted(ref.files) == sorted(mine.files)
    for k in ref.files:
        np.testing.assert_array_equal(ref[k], mine[k])
    assert [r.window for r in again] == [r.window for r in roms]


def test_version_mismatch_rejected(golden_dir, tmp_path):
    from paper_2310_04734_b200 import artifacts
    z = dict(np.load(golden_dir / "rom_ref.npz"))
    z["version"] = np.array(2)
    np.savez_compressed(tmp_path / "bad.npz", **z)
    with pytest.raises(ValueError):
        artifacts.load_roms(tmp_path / "bad.npz", _fom(golden_dir))


@pytest.mark.gpu
def test_sweep_of_reference_roms_reproduces_reference_frf(cuda, golden_dir, tmp_path):
    from paper_2310_04734_b200 import artifacts, mor
    roms = artifacts.load_roms(golden_dir / "rom_ref.npz", _fom(golden_dir))
    v = np.load(golden_dir / "frf_ref_values.npz")
    sw = mor.rom_sweep(roms, list(v["freqs"]))
    np.testing.assert_array_equal(sw.window_index, v["window_index"])
    np.testing.assert_allclose(np.array(sw.frf), v["frf"], rtol=1e-10)
    files = artifacts.write_sweep_artifacts(tmp_path, sw)
    assert files[0].name == "frf_mor.csv"
    lines = files[0].read_text().splitlines()
    ref = (golden_dir / "frf_ref.csv").read_text().splitlines()
    assert lines[0] == ref[0] and len(lines) == len(ref)
