"""B200-native QMoE compressed decode + matvec (drop-in for moepack's codec path).

The public surface mirrors the reference package `moepack`
(/root/reference/pkg/src/moepack/__init__.py): encode / decompress /
fused_matvec / simulate_warp_row over CompressedMatrix and the 65,536-entry
Dictionary, plus the device-resident pieces this build adds (DeviceMatrix,
the grouped MoE layer and expert-parallel layout). Every compute call goes
through libqmoe.so (sm_100a); importing fails if it is missing.
"""

from . import _lib  # noqa: F401  (fails loudly without libqmoe.so)
from .bf16 import bf16_bits_to_f32, bf16_round, f32_to_bf16_bits
from .codec import (
    CompressedMatrix,
    DeviceMatrix,
    SymbolTrace,
    WarpTrace,
    decompress,
    encode,
    encode_device,
    fused_matvec,
    pad_to_even,
    read_checkpoint,
    read_checkpoint_device,
    read_stacked_device,
    simulate_warp_row,
    write_checkpoint,
)
from .dictionary import (
    DEFAULT_P0,
    DICT_SIZE,
    MAX_PAIRS,
    Dictionary,
    PairDistribution,
    Trie,
    generate_dictionary,
    load_dictionary,
    pack_decode_words,
    save_dictionary,
    unpack_decode_words,
)
from .errors import ConfigError, CorruptionError, DictionaryMismatchError, MoepackError, TierCapacityError
from .moe import CompressedMoELayer, CompressedMoEModel, forward_stream, load_moe_layer
from .pipeline import DeviceRouter, RouterSim
from .quantize import QuantGrid, TernaryMatrix, make_grid, reconstruction_levels, rtn_quantize, rtn_quantize_device
from .stats import RateReport, compression_rate, natural_sparsity, sample_ternary, theoretical_limit

__all__ = [n for n in dir() if not n.startswith("_")]
