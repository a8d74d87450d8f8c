"""Minimal in-process two-party channel with the reference's endpoint API.

The reference's transport (transport.py) is outside the hot path; the
protocol functions in linprot.py only call `end.send(phase, payload)`,
`end.recv(phase)`, `end.recv_any()` and `end.stats.report()`, so they run
unchanged over the reference's ChannelEnd objects.  This module provides the
same surface (framing tag u8 + length u32, per-phase byte accounting, phase
checking, two-thread runner) for tests and benchmarks on the GPU box, where
the reference package is not installed.
"""
from __future__ import annotations

import queue
import struct
import threading

PHASE_SETUP, PHASE_OFFLINE, PHASE_ONLINE, PHASE_NONLINEAR = "setup", "offline", "online", "nonlinear"
PHASES = (PHASE_SETUP, PHASE_OFFLINE, PHASE_ONLINE, PHASE_NONLINEAR)
CLIENT, SERVER = "client", "server"
HEADER_BYTES = 5


class TransportError(Exception):
    pass


class ChannelClosedError(TransportError):
    pass


class PhaseMismatchError(TransportError):
    pass


class ChannelStats:
    def __init__(self, capture: bool = False):
        self._lock = threading.Lock()
        self.sent: dict = {}
        self.rounds = 0
        self._last = None
        self.capture = capture
        self.transcript = {CLIENT: bytearray(), SERVER: bytearray()}

    def record(self, sender: str, phase: str, frame: bytes):
        with self._lock:
            self.sent[(sender, phase)] = self.sent.get((sender, phase), 0) + len(frame)
            if self._last != sender:
                self.rounds += 1
                self._last = sender
            if self.capture:
                self.transcript[sender] += frame

    def report(self) -> dict:
        with self._lock:
            by_phase = {p: 0 for p in PHASES}
            for (_, p), v in self.sent.items():
                by_phase[p] += v
            return {
                "bytes_by_phase": by_phase,
                "bytes_client_to_server": sum(v for (s, _), v in self.sent.items() if s == CLIENT),
                "bytes_server_to_client": sum(v for (s, _), v in self.sent.items() if s == SERVER),
                "total_bytes": sum(self.sent.values()),
                "rounds": self.rounds,
            }


class ChannelEnd:
    def __init__(self, role: str, stats: ChannelStats, out_q, in_q, timeout: float):
        self.role, self.stats, self._out, self._in, self._timeout = role, stats, out_q, in_q, timeout

    def send(self, phase: str, payload: bytes):
        if phase not in PHASES:
            raise ValueError(f"unknown phase {phase!r}")
        payload = bytes(payload)
        self.stats.record(self.role, phase, struct.pack("<BI", PHASES.index(phase), len(payload)) + payload)
        self._out.put((PHASES.index(phase), payload))

    def _get(self):
        try:
            item = self._in.get(timeout=self._timeout)
        except queue.Empty:
            raise ChannelClosedError(f"{self.role} timed out waiting for a frame") from None
        if item is None:
            raise ChannelClosedError("peer closed the channel")
        return item

    def recv(self, expected_phase: str) -> bytes:
        tag, payload = self._get()
        if PHASES[tag] != expected_phase:
            raise PhaseMismatchError(f"{self.role} expected {expected_phase!r}, got {PHASES[tag]!r}")
        return payload

    def recv_any(self):
        tag, payload = self._get()
        return PHASES[tag], payload

    def close(self):
        self._out.put(None)


def inproc_pair(timeout: float = 600.0, capture: bool = False) -> tuple[ChannelEnd, ChannelEnd]:
    stats = ChannelStats(capture)
    c2s, s2c = queue.Queue(), queue.Queue()
    return ChannelEnd(CLIENT, stats, c2s, s2c, timeout), ChannelEnd(SERVER, stats, s2c, c2s, timeout)


def run_pair(client_fn, server_fn, client_end: ChannelEnd, server_end: ChannelEnd):
    """Run both parties concurrently (server on a thread); re-raise server errors."""
    result, error = {}, {}

    def _server():
        try:
            result["server"] = server_fn(server_end)
        except Exception as e:  # noqa: BLE001
            error["server"] = e

    th = threading.Thread(target=_server, daemon=True)
    th.start()
    try:
        result["client"] = client_fn(client_end)
    except Exception:
        th.join(timeout=5.0)
        if "server" in error:
            raise error["server"]
        raise
    th.join()
    if "server" in error:
        raise error["server"]
    return result["client"], result.get("server")
