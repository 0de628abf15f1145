"""Communication accounting mirroring the reference's CommStats (distsim.py:193-287).

The reference counts payload scalars per simulated message; here the same counts are
derived from the K1 outputs (participation masks and sample totals), and the real
bytes that crossed the interconnect are reported beside them.
"""
from __future__ import annotations

from dataclasses import dataclass, field as dc_field

SCALARS_PER_SAMPLE = 6  # distsim.py:59
SCALARS_PER_TILE_PACKET = 9  # distsim.py:60
COMPOSITOR = -1


@dataclass
class WorkerStats:
    scalars_sent: int = 0
    scalars_received: int = 0
    messages_sent: int = 0
    messages_received: int = 0


@dataclass
class CommStats:
    rays: int = 0
    participations: int = 0
    samples_assigned: int = 0
    workers: dict = dc_field(default_factory=dict)
    compositor: WorkerStats = dc_field(default_factory=WorkerStats)
    phase_seconds: dict = dc_field(default_factory=dict)
    link_bytes: int = 0  # bytes actually moved by the exchange collective

    def _party(self, pid: int) -> WorkerStats:
        if pid == COMPOSITOR:
            return self.compositor
        return self.workers.setdefault(pid, WorkerStats())

    def record(self, sender: int, receiver: int, scalars: int, messages: int = 1) -> None:
        s = self._party(sender)
        r = self._party(receiver)
        s.scalars_sent += scalars
        s.messages_sent += messages
        r.scalars_received += scalars
        r.messages_received += messages

    def add_time(self, phase: str, seconds: float) -> None:
        self.phase_seconds[phase] = self.phase_seconds.get(phase, 0.0) + seconds

    @property
    def scalars_sent_total(self) -> int:
        return sum(w.scalars_sent for w in self.workers.values()) + self.compositor.scalars_sent

    @property
    def scalars_received_total(self) -> int:
        return (sum(w.scalars_received for w in self.workers.values())
                + self.compositor.scalars_received)

    @property
    def messages_sent_total(self) -> int:
        return sum(w.messages_sent for w in self.workers.values()) + self.compositor.messages_sent

    def merge(self, other: "CommStats") -> None:
        """Accumulate another batch's counts (distsim.py:250-265): per-worker and compositor
        scalars / messages, ray and sample totals, phase times, link bytes."""
        self.rays += other.rays
        self.participations += other.participations
        self.samples_assigned += other.samples_assigned
        for pid, ws in list(other.workers.items()) + [(COMPOSITOR, other.compositor)]:
            mine = self._party(pid)
            mine.scalars_sent += ws.scalars_sent
            mine.scalars_received += ws.scalars_received
            mine.messages_sent += ws.messages_sent
            mine.messages_received += ws.messages_received
        for phase, sec in other.phase_seconds.items():
            self.add_time(phase, sec)
        self.link_bytes += other.link_bytes

    def samples_per_ray_mean(self) -> float:
        return self.samples_assigned / self.rays if self.rays else 0.0

    def samples_per_participation(self) -> float:
        return self.samples_assigned / self.participations if self.participations else 0.0


def stats_json(stats: CommStats, protocol: str, num_workers: int) -> dict:
    """Same document shape as distsim.stats_json (distsim.py:268-287)."""
    per_worker = []
    for tid in range(num_workers):
        ws = stats.workers.get(tid, WorkerStats())
        per_worker.append({"tile_id": tid, "scalars_sent": ws.scalars_sent,
                           "scalars_received": ws.scalars_received,
                           "messages_sent": ws.messages_sent})
    return {"protocol": protocol, "num_workers": num_workers, "rays": stats.rays,
            "scalars_sent_total": stats.scalars_sent_total, "per_worker": per_worker,
            "samples_per_ray_mean": stats.samples_per_ray_mean(),
            "link_bytes": stats.link_bytes}
