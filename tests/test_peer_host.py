"""Host-only layout check of peer-mapped halos (sldg_peer_halo_check): the pads
are mappings of the neighbours' edge chunks, so pad and layer chunks of both precision sections
must be whole allocation granules on every rank, and every rank needs >= 2 pad layers."""
import pytest

from paper_1603_07008_b200 import SldgError
from paper_1603_07008_b200.sldg import peer_halo_check

MiB = 1 << 20


def test_c5_layout_accepted_at_every_bench_world_size():
    # C5: 128^3 cells per layer -> 16 MiB fp64 + 64 MiB fp32 per layer (k = 3 mixed)
    for world in (1, 2, 4, 8):
        assert peer_halo_check([128] * 4, 3, "mixed", world, 2, 2 * MiB) is None
    assert peer_halo_check([128] * 4, 3, "fp64", 8, 2, 2 * MiB) is None


def test_too_few_layers_per_rank():
    why = peer_halo_check([128] * 4, 3, "mixed", 64, 2, 2 * MiB)  # 2 layers per rank < 2 pad
    assert why and "2 * pad" in why
    # an uneven split: the smaller ranks decide
    assert peer_halo_check([128, 128, 128, 9], 3, "mixed", 2, 2, 2 * MiB) is None  # 5 / 4 layers
    assert peer_halo_check([128, 128, 128, 9], 3, "mixed", 2, 3, 2 * MiB) is not None  # 4 < 6


def test_granularity_of_each_section():
    # 32^4 k = 2 mixed: fp64 layer 256 KiB, fp32 layer 15 * 128 KiB = 1.875 MiB
    assert "fp32 section" in peer_halo_check([32] * 4, 2, "mixed", 1, 8, 2 * MiB)
    assert peer_halo_check([32] * 4, 2, "mixed", 1, 16, 2 * MiB) is None
    # pad 8 passes the fp64 section alone (fp64 storage: 16 * 256 KiB = 4 MiB per layer)
    assert peer_halo_check([32] * 4, 2, "fp64", 1, 1, 2 * MiB) is None
    # fp64 section too small: 32 * 32 cells * 8 B = 8 KiB per layer, 32 KiB per 4-layer pad
    assert "fp64 section" in peer_halo_check([32, 32, 16], 1, "fp64", 1, 4, 2 * MiB)
    # a 32 KiB granule accepts what 2 MiB (and 64 KiB) refuse
    assert peer_halo_check([32, 32, 16], 1, "fp64", 1, 4, 32 << 10) is None
    assert peer_halo_check([32, 32, 16], 1, "fp64", 1, 4, 64 << 10) is not None


def test_bad_arguments():
    with pytest.raises(SldgError, match="EINVAL"):
        peer_halo_check([32] * 4, 2, "mixed", 0, 2)
    with pytest.raises(SldgError, match="EINVAL"):
        peer_halo_check([32, 32, 4], 2, "mixed", 8, 2)  # extent < world
    assert "D >= 2" in peer_halo_check([1024], 2, "mixed", 1, 2)
