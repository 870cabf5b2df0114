"""Host-side launch planning of the engine (no GPU): the weight-gradient launch chunks of a layer
(<= 16 problems per grouped launch, every logical rank exactly once, balanced, the one-GPU plan's
error-compression slot pairs in the first launch) and the layer-0 compressor-gradient batch split
(one round of 1-SM tiles on 148 SMs, whole 128-row K blocks)."""
import pytest

from paper_2508_00960_b200 import schedule
from paper_2508_00960_b200.errors import ConfigurationError


@pytest.mark.parametrize("R,p", [(8, 8), (4, 4), (2, 2), (4, 8), (2, 8), (1, 8), (6, 6), (16, 16)])
@pytest.mark.parametrize("nprob", [1, 2, 3])
@pytest.mark.parametrize("with_errors", [False, True])
def test_wgrad_chunks_cover_ranks_within_launch_limit(R, p, nprob, with_errors):
    if with_errors and (p // 2 + nprob > schedule.MAX_PROBS):
        with pytest.raises(ConfigurationError):
            schedule.wgrad_launch_chunks(R, p, nprob, R, with_errors)
        return
    chunks = schedule.wgrad_launch_chunks(R, p, nprob, R, with_errors)
    covered = [j for c0, c1 in chunks for j in range(c0, c1)]
    assert covered == list(range(R))
    for i, (c0, c1) in enumerate(chunks):
        probs = nprob * (c1 - c0) + (p // 2 if with_errors and i == 0 else 0)
        assert 1 <= c1 - c0 and probs <= schedule.MAX_PROBS, (chunks, i, probs)
    sizes = [c1 - c0 for c0, c1 in chunks]
    assert max(sizes) - min(sizes) <= max(1, R // len(chunks)), sizes


def test_wgrad_chunks_c3_one_gpu():
    """C3 on one GPU (R = p = 8): two launches of 4 ranks per inner layer; with the error
    compression the first holds 4 pair problems + 12 weight-gradient problems = 16."""
    assert schedule.wgrad_launch_chunks(8, 8, 3, 8, False) == [(0, 4), (4, 8)]
    assert schedule.wgrad_launch_chunks(8, 8, 3, 8, True) == [(0, 4), (4, 8)]
    assert schedule.wgrad_launch_chunks(8, 8, 2, 8, True) == [(0, 4), (4, 8)]   # top layer: balanced
    assert schedule.wgrad_launch_chunks(8, 8, 2, 1, False) == [(j, j + 1) for j in range(8)]


@pytest.mark.parametrize("n_items,k,s,batch,expect", [
    (1, 128, 2048, 8192, 16),     # C3, one logical rank per launch: 8 tiles -> 128
    (2, 128, 2048, 8192, 8),      # two ranks per GPU (N = 4)
    (8, 128, 2048, 8192, 2),      # one GPU, all 8 ranks: 64 tiles -> 128
    (4, 32, 128, 512, 4),         # the engine test shape
    (4, 32, 128, 64, 1),          # batch too small for 128-row chunks
    (1, 256, 8192, 8192, 2),      # C4 per rank: 64 tile-equivalents -> 128
])
def test_layer0_split(n_items, k, s, batch, expect):
    nsplit = schedule.layer0_split(n_items, k, s, batch)
    assert nsplit == expect
    tiles = n_items * -(-k // 128) * -(-s // 256)
    assert tiles * nsplit <= 148 or nsplit == 1
    assert batch % nsplit == 0 and (nsplit == 1 or (batch // nsplit) % 128 == 0)
    assert n_items * nsplit <= schedule.MAX_PROBS


@pytest.mark.parametrize("knob", ["PPX_NO_SPLITK", "PPX_NO_K3G", "PPX_AB_TF32_HI_COPY", "PPX_DEBUG_EPI", "PPX_QBAL"])
def test_bench_refuses_plan_knobs(knob, monkeypatch):
    """The bench line is always the default plan: every A/B or debug switch is refused."""
    import bench
    monkeypatch.setenv(knob, "1")
    with pytest.raises(SystemExit):
        bench.refuse_debug_knobs()


def test_bench_allows_library_path(monkeypatch):
    import bench
    for k in [k for k in list(__import__("os").environ) if k.startswith("PPX_")]:
        monkeypatch.delenv(k, raising=False)
    monkeypatch.setenv("PPX_NO_NUMA_BIND", "1")
    monkeypatch.setenv("PPX_LIB", "/tmp/libppx.so")
    bench.refuse_debug_knobs()
