"""DMA-buffer rollback and the ordered failover chain.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

P:36 (§4.3 Technique II): "After receiving an OOB failure notification, the
sender rewinds to the first chunk without a completion, and the receiver
resets to the last confirmed chunk.  The system retransmits all subsequent
chunks over the selected backup NIC.  If that NIC later fails, R²CCL moves to
the next NIC in the failover chain and retransmits from the same rollback
point."  SPEC S:243-251 (rollback op), S:252-260 (migrate op).

P:27 (§4.3 Technique I): "R²CCL also orders backup NICs by PCIe distance,
activating the closest healthy NIC during migration.  The ordered NIC chain
supports successive failovers."  On NVSwitch every channel of a peer is at the
same distance; reading C-2 orders the backups of channel c by forward cyclic
channel distance c+1, c+2, ... (ties by id).

Reading C-4/C-5: a completion is the flag word in the receiver's memory, so
sender_resume = first position without a flag and receiver_floor = end of the
contiguous confirmed prefix = sender_resume - 1.  Reading C-7: exactly the
positions without a completion are retransmitted (re-evaluated at every
failover).
"""
from __future__ import annotations


class NoBackup(Exception):
    """The failover chain is exhausted (S:256 'NoBackup if chain exhausted')."""


class NoFailurePending(Exception):
    """rollback() called with no failure pending."""


def rollback(completed: list[bool], failure_pending: bool = True) -> tuple[int, int]:
    """(sender_resume, receiver_floor) from a connection's completion ledger.

    sender_resume = min{q : not completed[q]} (len if all complete);
    receiver_floor = max{q : completed[0..q] all confirmed} (-1 if none).
    """
    if not failure_pending:
        raise NoFailurePending("rollback called with no failure pending")
    resume = len(completed)
    for q, done in enumerate(completed):
        if not done:
            resume = q
            break
    floor = resume - 1
    return resume, floor


def residual(completed: list[bool]) -> list[int]:
    """Positions to retransmit: exactly those without a completion (C-7)."""
    return [q for q, done in enumerate(completed) if not done]


def failover_chain(channel: int, K: int) -> list[int]:
    """Backups of `channel`, closest first: c+1, c+2, ..., c+K-1 (mod K)."""
    return [(channel + d) % K for d in range(1, K)]


def failover_chain_by_distance(distances: dict[int, int]) -> list[int]:
    """S:45-53 generic form: sort ascending by distance, ties by id."""
    return sorted(distances, key=lambda nic: (distances[nic], nic))


def migrate(chain: list[int], healthy: set[int]) -> tuple[int, int]:
    """First healthy entry of the chain -> (channel, chain position).

    Raises NoBackup when every chain entry has failed.
    """
    for pos, c in enumerate(chain):
        if c in healthy:
            return c, pos
    raise NoBackup("failover chain exhausted")
