"""Topology discovery for the synthesis target.

The reference "probes the target hardware topology" and
names topologies in the schedule file.  On an 8xB200 box
every GPU reaches every other through NVSwitch at the full per-GPU NVLink 5
bandwidth, so the synthesis target moves from the DGX-1 hybrid cube-mesh to
``switch:N`` (per-GPU egress/ingress groups); ``full:N`` is
the per-pair logical view.  This probes NVML (NVLink state and remote device
types) and CUDA peer access and returns the target name plus the evidence.
"""
from __future__ import annotations

from typing import Dict, List, Optional


def _nvml_links(ndev: int) -> Optional[List[Dict]]:
    try:
        import pynvml as nv
    except ImportError:
        return None
    try:
        nv.nvmlInit()
    except Exception:
        return None
    out = []
    try:
        for i in range(ndev):
            h = nv.nvmlDeviceGetHandleByIndex(i)
            links = {"active": 0, "to_switch": 0, "to_gpu": 0}
            for link in range(getattr(nv, "NVML_NVLINK_MAX_LINKS", 18)):
                try:
                    if nv.nvmlDeviceGetNvLinkState(h, link) != nv.NVML_FEATURE_ENABLED:
                        continue
                except Exception:
                    continue
                links["active"] += 1
                try:
                    t = nv.nvmlDeviceGetNvLinkRemoteDeviceType(h, link)
                    if t == getattr(nv, "NVML_NVLINK_DEVICE_TYPE_SWITCH", 2):
                        links["to_switch"] += 1
                    elif t == getattr(nv, "NVML_NVLINK_DEVICE_TYPE_GPU", 0):
                        links["to_gpu"] += 1
                except Exception:
                    pass
            out.append(links)
    finally:
        try:
            nv.nvmlShutdown()
        except Exception:
            pass
    return out


def discover(ndev: Optional[int] = None) -> Dict:
    """{'target': 'switch:N' | 'full:N' | 'loopback:1' | 'unknown', ...evidence}."""
    try:
        import torch
        cuda = torch.cuda.is_available()
        n = ndev if ndev is not None else (torch.cuda.device_count() if cuda else 0)
    except Exception:
        cuda, n = False, 0
    info: Dict = {"devices": n}
    if n == 0:
        info["target"] = "unknown"
        return info
    import torch
    peer = [[i == j or torch.cuda.can_device_access_peer(i, j) for j in range(n)] for i in range(n)]
    info["peer_access"] = peer
    links = _nvml_links(n)
    info["nvlink"] = links
    if n == 1:
        info["target"] = "loopback:1"
    elif all(all(r) for r in peer):
        through_switch = links is not None and all(l["to_switch"] > 0 for l in links)
        info["target"] = f"switch:{n}" if through_switch else f"full:{n}"
    else:
        info["target"] = "unknown"
    return info
