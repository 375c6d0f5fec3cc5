"""Loading of the golden fixtures written by tests/golden/make_golden.py."""
from __future__ import annotations

from pathlib import Path

import numpy as np

from paper_1810_03931_b200 import abi, models

GOLDEN = Path(__file__).resolve().parent / "golden"

_BY_ID = {
    abi.MODEL_DUFFING: lambda k: models.DuffingSystem(),
    abi.MODEL_DUFFING_MAX_ACCESSORY: lambda k: models.DuffingMaxAccessorySystem(),
    abi.MODEL_DUFFING_MAX_EVENT: lambda k: models.DuffingMaxEventSystem(k[0], int(k[1])),
    abi.MODEL_DUFFING_MAXMIN: lambda k: models.DuffingMaxMinSystem(),
    abi.MODEL_KELLER_MIKSIS: lambda k: models.KellerMiksisSystem(),
    abi.MODEL_BUBBLE_COLLAPSE: lambda k: models.BubbleCollapseSystem(k[0]),
    abi.MODEL_VALVE: lambda k: models.ValveSystem(k[0]),
    abi.MODEL_DUFFING_LYAPUNOV: lambda k: models.DuffingLyapunovSystem(),
    abi.MODEL_CONSTANT: lambda k: models.ConstantDef(k[0]),
    abi.MODEL_CUBIC_TIME: lambda k: models.CubicTimeDef(),
    abi.MODEL_EXPONENTIAL: lambda k: models.ExponentialDef(),
    abi.MODEL_UNIT_SLOPE: lambda k: models.UnitSlopeDef(),
    abi.MODEL_COUNTING: lambda k: models.CountingDef(),
    abi.MODEL_RAMP: lambda k: models.RampDef(k[0], k[1], int(k[2]), int(k[3]), k[4], int(k[5])),
    abi.MODEL_DECAY: lambda k: models.DecayDef(),
    abi.MODEL_SEAT_CONTACT: lambda k: models.SeatContactDef(),
    abi.MODEL_HARMONIC: lambda k: models.HarmonicDef(),
    abi.MODEL_BLOWUP: lambda k: models.BlowUpDef(),
}


def fixture_names():
    return sorted(p.stem for p in GOLDEN.glob("*.npz"))


def load(name: str) -> dict:
    z = np.load(GOLDEN / f"{name}.npz")
    d = {k: z[k] for k in z.files}
    d["model"] = _BY_ID[int(d["model_id"])]([float(v) for v in d["consts"]])
    d["name"] = name
    return d


def outcome_bytes(o: np.ndarray) -> np.ndarray:
    """Outcome records without the 7 padding bytes (for bitwise compares)."""
    raw = np.ascontiguousarray(o).view(np.uint8).reshape(-1, 56)
    keep = [i for i in range(56) if not 9 <= i < 16]
    return raw[:, keep]
