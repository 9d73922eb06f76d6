"""Parity at BASELINE.json's full sizes, through the same C-ABI entry points
bench.py times (machinery and checks: tests/fullsize_common.py):
* config[1] = C2, the bench.py N=1 workload: N = 1024^2 values x 2048,
  4 heads, k = 32, 16K tokens, bf16, Memory+ gate;
* config[2] = C3 at G = 1: N = 4096^2 values x 2048 (a 64 GiB table; fits
  one B200), same layer shape.
"""
import pytest
import torch

from tests.fullsize_common import Full

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module", params=["c2", "c3"])
def case(request):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    f = Full(request.param)
    run = f.run()
    return f, run, f.host_tables()


def test_sampled_tokens(case):
    f, run, tb = case
    f.check_sampled_tokens(run, tb)


def test_sampled_value_rows(case):
    f, run, tb = case
    f.check_sampled_value_rows(run, tb)


def test_key_gradient_identity(case):
    f, run, tb = case
    f.check_key_gradient_identity(run, tb)


def test_row_set_properties(case):
    f, run, tb = case
    f.check_row_set(run)
