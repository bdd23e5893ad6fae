"""Measured selection (tune.py): the table construction is pure host logic
(CPU); World.tune / Communicator.tune on the GPUs are in
tests/test_gpu_collectives.py and tests/test_gpu_multiprocess.py."""

import pytest

from paper_2504_09014_b200 import _lib
from paper_2504_09014_b200.errors import NoAlgoError
from paper_2504_09014_b200.tune import algo_id, nvls_min_from_times, selection_from_times

K = 1024


def test_fastest_per_size_runs_merged():
    sizes = [K, 4 * K, 16 * K, 64 * K, 256 * K]
    times = {"1pa": [1.0, 1.1, 2.0, None, None],     # beyond the LL capacity from 64 KiB
             "2pa": [3.0, 3.0, 1.5, 1.6, 2.0],
             "1pa_hb": [1.2, 1.0, 1.8, 1.7, 3.0]}
    assert selection_from_times(sizes, times) == [(K, "1pa"), (4 * K, "1pa_hb"), (256 * K, "2pa")]


def test_unsorted_sizes_and_single_winner():
    sizes = [64 * K, K]
    times = {"2pa": [1.0, 1.0], "1pa": [None, 2.0]}
    # sizes are sorted first; the time lists follow the sorted order
    assert selection_from_times(sizes, times) == [(64 * K, "2pa")]


def test_nvls_min_is_the_start_of_the_winning_tail():
    sizes = [K, 64 * K, K * K, 16 * K * K]
    assert nvls_min_from_times(sizes, [5, 1, 9, 1], [4, 2, 3, 2]) == 16 * K * K   # wins, loses, wins
    assert nvls_min_from_times(sizes, [5, 1, 1, 1], [4, 2, 3, 2]) == 64 * K
    assert nvls_min_from_times(sizes, [5, 5, 5, 5], [4, 2, 3, 2]) is None


def test_algo_ids():
    assert algo_id("2pa_ll") == _lib.ALGOS["2pa_ll"]
    assert algo_id("ring_ag+ring") == _lib.ALGOS["ring_ag"] | _lib.CF_ALGO_RING_LINKS
    with pytest.raises(NoAlgoError):
        algo_id("auto")
    with pytest.raises(NoAlgoError):
        algo_id("2ph")


def test_package_exports_the_reference_surface():
    """Every name of the reference's ``__all__`` (cf/__init__.py:12-17) imports
    from the drop-in package; transfer_time keeps the reference's alpha-beta
    definition (cf/timing.py:48-51)."""
    import paper_2504_09014_b200 as pkg
    ref_all = ["CostParams", "ExecutionPlan", "LoweringParams", "ProgramGraph", "Runtime", "RunResult",
               "Selector", "SimWorld", "algobw", "collective", "lower", "make_world", "parse_plan",
               "run_benchmark", "select_algorithm", "serialize_plan", "simulate_timed", "transfer_time",
               "validate_plan"]
    for name in ref_all:
        assert hasattr(pkg, name) and name in pkg.__all__, name
    p = pkg.CostParams()
    assert pkg.transfer_time("intra", 1 << 20, p) == pytest.approx(829e-9 + (1 << 20) / 397.5e9)
    assert pkg.transfer_time("inter", 1000, p) == pytest.approx(4.89e-6 + 1000 / 48.94e9)


def test_channel_objects_validate_like_the_reference():
    """cf/channels.py:159-160: an unknown protocol is E_WRONG_PROTOCOL (raised
    before any device work)."""
    from paper_2504_09014_b200.channels import MemoryChannel
    from paper_2504_09014_b200.errors import WrongProtocolError
    with pytest.raises(WrongProtocolError):
        MemoryChannel(None, None, "LL128", 0, 1)
