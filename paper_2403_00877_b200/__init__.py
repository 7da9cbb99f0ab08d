"""B200-native DMT / SPTT hot path (arXiv 2403.00877).

Drop-in for the reference ``towersim`` API on the SPTT path: the same names,
signatures and exceptions (tower_exchange, baseline_exchange, realign,
TowerPlan, ExchangeOptions, TMConfig, tm_forward, shard_tables, ...) backed by
sm_100a CUDA kernels in libdmt.so (C ABI: include/dmt.h) and NCCL.  There is
no CPU fallback.
"""

from .embedding import (
    COLUMN_WISE,
    POOL_MEAN,
    POOL_NONE,
    POOL_SUM,
    ROW_WISE,
    TABLE_WISE,
    EmbeddingTable,
    Shard,
    ShardedEmbedding,
    SparseBatch,
    TablePlan,
    init_table_deterministic,
    load_table_csv,
    lookup,
    make_batch,
    shard_tables,
    split_ranges,
)
from .errors import (
    ConfigError,
    ConstraintError,
    DomainError,
    EquivalenceError,
    IngestionError,
    LayoutError,
    NumericError,
    PlanError,
    ProtocolError,
    ReportError,
    ShapeError,
    TableLookupError,
    TowersimError,
)
from .exchange import (
    ExchangeOptions,
    ExchangeResult,
    OutputLayout,
    TowerPlan,
    baseline_exchange,
    realign,
    tower_exchange,
)
from .simnet import CommTrace
from .topology import (
    ClusterTopology,
    TowerLayout,
    class_members,
    class_order,
    link_class,
    peer_order,
    peers,
)
from .towermod import (
    DCNWeights,
    DLRMWeights,
    TMConfig,
    TowerModule,
    balanced_group_sizes,
    compression_ratio,
    crossnet_layer,
    init_tm_weights,
    interaction_pairs,
    tm_dcn_forward,
    tm_dlrm_forward,
    tm_flops,
    tm_forward,
    tm_output_width,
)

__version__ = "0.1.0"
