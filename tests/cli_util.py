"""Helpers for the djg command-line tool tests (mirrors the reference's
tests/test_cli.cpp fixtures)."""
import subprocess
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
CLI = ROOT / "paper_2106_14189_b200" / "_build" / "djg"


def run_cli(*args, cwd=None):
    p = subprocess.run([str(CLI), *map(str, args)], capture_output=True, text=True, cwd=cwd, timeout=600)
    return p.returncode, p.stdout, p.stderr


def tiny_run_config(d: Path, engine: str = "djtled", extra: str = "") -> str:
    """tiny_run_config of test_cli.cpp:41-48."""
    return ("[mesh]\ngenerate = box\nkind = T4\nextent = 0.1\ndivisions = 2 2 2\n"
            "[material]\nmodel = NH\nmu = 6567\nkappa = 326210\nrho = 1060\n"
            "[bc]\nfix = zmin all\nprescribe = zmax z 0.005 0.02\n"
            "[time]\ndt = auto\nsafety = 0.8\nt_end = 0.02\nalpha = 100\n"
            f"[run]\nengine = {engine}\nthreads = 1\n"
            f"[output]\nfield = {d}/out.vtk\nreport = {d}/report.txt\n" + extra)


def write(path: Path, text: str) -> Path:
    path.write_text(text)
    return path


def read_report(path: Path) -> dict:
    out = {}
    for line in path.read_text().splitlines():
        parts = line.split(" ", 1)
        if len(parts) == 2:
            out[parts[0]] = parts[1]
    return out


def read_vtk_field(path: Path, dtype) -> np.ndarray:
    text = path.read_text()
    tail = text[text.index("VECTORS displacement"):].split("\n", 1)[1]
    return np.array(tail.split(), dtype=np.float64).astype(dtype)
