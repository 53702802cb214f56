"""Transport layer: the contract plus the ``sim``, ``socket`` and ``nvlink`` kinds.

``transport_init`` is the plug-in boundary of the reference
(``pkg/src/commshim/transport/__init__.py:42-76``); ``kind="nvlink"`` selects
the B200 transport backed by ``libm4d.so``.
"""

from __future__ import annotations

from ..errors import ConfigurationError
from .base import (
    DEFAULT_MAX_COUNT,
    MAX_TAG,
    RESERVED_TAG_LIMIT,
    WORLD_CHANNEL,
    DeviceRegion,
    DeviceView,
    LinkModel,
    MemoryDomain,
    Transport,
    TransportConfig,
    TransportMetrics,
    TransferRequest,
    as_view,
)
from .sim import SimFabric, SimTransport

__all__ = [
    "DEFAULT_MAX_COUNT",
    "DeviceRegion",
    "DeviceView",
    "LinkModel",
    "MAX_TAG",
    "MemoryDomain",
    "NvlinkTransport",
    "RESERVED_TAG_LIMIT",
    "SimFabric",
    "SimTransport",
    "SocketTransport",
    "Transport",
    "TransportConfig",
    "TransportMetrics",
    "TransferRequest",
    "WORLD_CHANNEL",
    "as_view",
    "transport_init",
]


def _init_sim(world_size: int, rank: int, config: TransportConfig) -> Transport:
    fabric = config.fabric
    if fabric is None:
        fabric = SimFabric(world_size, link=config.link, max_count=config.max_count,
                           device_aware=config.device_aware)
    if fabric.world_size != world_size:
        raise ConfigurationError(f"fabric world size {fabric.world_size} != requested {world_size}")
    return fabric.transport(rank)


def _init_socket(world_size: int, rank: int, config: TransportConfig) -> Transport:
    from .tcp import SocketTransport

    if config.rank_map is None:
        raise ConfigurationError("socket transport requires a rank -> (host, port) map")
    return SocketTransport(world_size, rank, config.rank_map, max_count=config.max_count,
                           device_aware=config.device_aware, connect_timeout=config.connect_timeout)


def _init_nvlink(world_size: int, rank: int, config: TransportConfig) -> Transport:
    from .nvlink import NvlinkTransport

    return NvlinkTransport(world_size, rank, config)


_KINDS = {"sim": _init_sim, "socket": _init_socket, "nvlink": _init_nvlink}


def transport_init(world_size: int, self_rank: int, config: TransportConfig) -> Transport:
    """Bring up this rank's transport of the configured kind and return it.

    ``sim`` worlds share the ``SimFabric`` in ``config.fabric`` (a private one is
    created when omitted); ``socket`` needs ``config.rank_map``; ``nvlink`` needs
    every rank of the world on one node and finds its peers through
    ``config.session`` (shared memory), see :mod:`.nvlink`.
    """
    init = _KINDS.get(config.kind)
    if init is None:
        raise ConfigurationError(f"unknown transport kind {config.kind!r}")
    return init(world_size, self_rank, config)


def __getattr__(name: str):
    if name == "SocketTransport":
        from .tcp import SocketTransport

        return SocketTransport
    if name == "NvlinkTransport":
        from .nvlink import NvlinkTransport

        return NvlinkTransport
    raise AttributeError(name)
