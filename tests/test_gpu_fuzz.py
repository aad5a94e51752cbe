"""Seeded randomised parity sweep on the CUDA path (see tests/_fuzz_cases.py)."""
import pytest

from _fuzz_cases import run_cases

pytestmark = pytest.mark.gpu


def test_random_cases_vs_oracle():
    assert run_cases(90, seed=20260810) == []


def test_random_cases_vs_oracle_warp_specialised_sweep():
    assert run_cases(50, seed=5128, variant=2) == []
