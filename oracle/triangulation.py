"""Emulated zero-byte probes and three-point triangulation.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

P:16 (§4.2): "both endpoints and an auxiliary NIC issue zero-byte RDMA Writes
as probes ... generating completions without payloads or receiver
involvement."  P:19: "A failed NIC produces immediate local probe errors,
while its peer observes timeouts; a broken link yields timeouts at both
endpoints, with the auxiliary NIC distinguishing single-endpoint vs.
dual-endpoint impairment."  SPEC S:314-337 (probe / triangulate)
(totality), S:356 (2-node: migrate anyway), S:368 (two local errors).

Reading C-11 (emulated outcome): probe(P -> Q, c) = LOCAL_ERROR if P's
endpoint on c failed; else TIMEOUT if Q's endpoint on c or a ring link
between P and Q on c failed; else SUCCESS.

Reading C-10 (decision table, first match wins):
 (1) L,L -> TWO_LOCAL            (2) pAB = L -> LOCAL_ENDPOINT(A)
 (3) pBA = L -> REMOTE_ENDPOINT(B)   (4) S,S -> NONE
 (5) exactly one T, other S -> LINK(A,B)
 (6) T,T, no aux -> INCONCLUSIVE (migrate anyway)
 (7) T,T & aux S,S -> LINK     (8) aux T,S -> ENDPOINT_UNREACHABLE(A)
 (9) aux S,T -> ENDPOINT_UNREACHABLE(B)  (10) aux T,T -> DUAL_ENDPOINT
 (11) any aux L -> INCONCLUSIVE (aux itself faulty).
Reading C-12: aux = lowest rank not in {A, B}, same channel.
"""
from __future__ import annotations

SUCCESS, LOCAL_ERROR, TIMEOUT = "S", "L", "T"
OUTCOMES = (SUCCESS, LOCAL_ERROR, TIMEOUT)

NONE = "NONE"
LOCAL_ENDPOINT = "LOCAL_ENDPOINT"
REMOTE_ENDPOINT = "REMOTE_ENDPOINT"
LINK = "LINK"
ENDPOINT_UNREACHABLE_A = "ENDPOINT_UNREACHABLE_A"
ENDPOINT_UNREACHABLE_B = "ENDPOINT_UNREACHABLE_B"
DUAL_ENDPOINT = "DUAL_ENDPOINT"
TWO_LOCAL = "TWO_LOCAL"
INCONCLUSIVE = "INCONCLUSIVE"
VERDICTS = (NONE, LOCAL_ENDPOINT, REMOTE_ENDPOINT, LINK, ENDPOINT_UNREACHABLE_A,
            ENDPOINT_UNREACHABLE_B, DUAL_ENDPOINT, TWO_LOCAL, INCONCLUSIVE)


def aux_rank(a: int, b: int, n: int) -> int | None:
    """Lowest rank not in {a, b} (C-12); None for a 2-rank ring."""
    for r in range(n):
        if r not in (a, b):
            return r
    return None


def link_dead_between(p: int, q: int, c: int, n: int, link_dead) -> bool:
    """Is a ring link between p and q on channel c dead?  link_dead[r][c] is
    the ring edge r -> r+1 (a cable fault kills both directions)."""
    return (q == (p + 1) % n and link_dead[p][c]) or (p == (q + 1) % n and link_dead[q][c])


def probe(p: int, q: int, c: int, n: int, ep_dead, link_dead) -> str:
    """Emulated probe outcome (C-11)."""
    if ep_dead[p][c]:
        return LOCAL_ERROR
    if ep_dead[q][c] or link_dead_between(p, q, c, n, link_dead):
        return TIMEOUT
    return SUCCESS


def triangulate(p_ab: str, p_ba: str, p_xa: str | None = None, p_xb: str | None = None) -> str:
    """Decision table C-10 (total over 3^2 and 3^4 outcomes)."""
    has_aux = p_xa is not None
    if has_aux and p_xb is None:
        raise ValueError("missing aux->B outcome (S:333)")
    if p_ab == LOCAL_ERROR and p_ba == LOCAL_ERROR:
        return TWO_LOCAL
    if p_ab == LOCAL_ERROR:
        return LOCAL_ENDPOINT
    if p_ba == LOCAL_ERROR:
        return REMOTE_ENDPOINT
    if p_ab == SUCCESS and p_ba == SUCCESS:
        return NONE
    if (p_ab, p_ba) in ((TIMEOUT, SUCCESS), (SUCCESS, TIMEOUT)):
        return LINK
    # both timed out
    if not has_aux:
        return INCONCLUSIVE
    if LOCAL_ERROR in (p_xa, p_xb):
        return INCONCLUSIVE
    if p_xa == SUCCESS and p_xb == SUCCESS:
        return LINK
    if p_xa == TIMEOUT and p_xb == SUCCESS:
        return ENDPOINT_UNREACHABLE_A
    if p_xa == SUCCESS and p_xb == TIMEOUT:
        return ENDPOINT_UNREACHABLE_B
    return DUAL_ENDPOINT


def run_round(a: int, b: int, c: int, n: int, ep_dead, link_dead) -> dict:
    """One triangulation round for connection (a -> b, c)."""
    x = aux_rank(a, b, n)
    out = [probe(a, b, c, n, ep_dead, link_dead), probe(b, a, c, n, ep_dead, link_dead)]
    if x is not None:
        out += [probe(x, a, c, n, ep_dead, link_dead), probe(x, b, c, n, ep_dead, link_dead)]
        v = triangulate(*out)
    else:
        v = triangulate(out[0], out[1])
    return {"verdict": v, "a": a, "b": b, "aux": x, "channel": c, "outcomes": tuple(out)}


def dead_after_verdict(v: str, a: int, b: int) -> tuple[list[int], bool]:
    """Which endpoints (ranks) a verdict condemns on its channel, and whether
    the link a->b is condemned (reading C-14; INCONCLUSIVE -> migrate the
    connection anyway)."""
    if v in (LOCAL_ENDPOINT, ENDPOINT_UNREACHABLE_A):
        return [a], False
    if v in (REMOTE_ENDPOINT, ENDPOINT_UNREACHABLE_B):
        return [b], False
    if v in (DUAL_ENDPOINT, TWO_LOCAL):
        return [a, b], False
    if v in (LINK, INCONCLUSIVE):
        return [], True
    return [], False


def reprobe_readmits(a: int, b: int, c: int, n: int, ep_dead, link_dead) -> bool:
    """"R²CCL also periodically reprobes to detect component recovery
    (e.g., NIC resets, cable fixes)".  A re-probe of the dead connection
    (A -> B, c) is an ordinary round (run_round); the connection is usable
    again exactly when the round finds nothing wrong, i.e. the verdict is NONE
    (A->B and B->A both succeed: both endpoints and the link between them are
    alive, reading C-11)."""
    return run_round(a, b, c, n, ep_dead, link_dead)["verdict"] == NONE
