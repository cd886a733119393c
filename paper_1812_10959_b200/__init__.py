"""paper_1812_10959_b200 — B200-native Dynamic Itemset Counting support count.

A drop-in for the DIC hot path of the reference ``dicmine`` package
(/root/reference/pkg/src/dicmine, arXiv 1812.10959): the transaction bitmap,
the per-chunk support count, the checkpoint state machine with candidate
generation/subset pruning, and multi-GPU sharding.  The public names below
keep the reference's signatures (dicmine/__init__.py:68-121, hot-path
subset); the arithmetic runs in hand-written sm_100a kernels
(lib/libdicb200.so, C ABI in include/dic_b200.h).  There is no CPU fallback.
"""

from .bitmap import MAX_ITEMS, BitDatabase, database_from_transactions
from .bits import cardinality, contains, encode_transaction, immediate_subsets, items_of, join, popcounts
from .catalog import LEGAL_TRANSITIONS, CountedItemset, ItemsetCatalog, Shape, TransitionAudit
from .config import MiningParams, absolute_support, default_interval
from .exceptions import (CorrectnessFailure, DicmineError, EmptyDatabase, FormatError, ItemOutOfRange,
                         ParseError, SpecError, UniverseTooLarge)
from .miner import mine_parallel, mine_serial, run_engine
from .phases import (FrequentItemset, MiningResult, MiningStats, check_full_pass, count_support_interval,
                     first_pass, make_candidates, prune)
from .sharding import ShardPlan
from .datasets import (LoadReport, item_frequencies, load_bitdb, load_transactions, load_transactions_with_report,
                       parse_transactions, save_bitdb, save_transactions, sniff_format)
from .estimator import DicMiner, as_bit_database, resolve_thread_count

__version__ = "0.1.0"

__all__ = [
    "MAX_ITEMS", "BitDatabase", "CorrectnessFailure", "CountedItemset", "DicmineError", "EmptyDatabase",
    "FormatError", "FrequentItemset", "ItemOutOfRange", "ItemsetCatalog", "LEGAL_TRANSITIONS", "MiningParams",
    "MiningResult", "MiningStats", "ParseError", "Shape", "ShardPlan", "SpecError", "TransitionAudit",
    "UniverseTooLarge", "absolute_support", "cardinality", "check_full_pass", "contains",
    "count_support_interval", "database_from_transactions", "default_interval", "encode_transaction",
    "first_pass", "immediate_subsets", "items_of", "join", "make_candidates", "mine_parallel", "mine_serial",
    "popcounts", "prune", "run_engine",
    "DicMiner", "LoadReport", "as_bit_database", "item_frequencies", "load_bitdb", "load_transactions",
    "load_transactions_with_report", "parse_transactions", "resolve_thread_count", "save_bitdb",
    "save_transactions", "sniff_format",
]
