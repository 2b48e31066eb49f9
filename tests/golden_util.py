"""Size-independent summaries of long trajectories (test infrastructure)."""
import numpy as np

_MASK = (1 << 64) - 1


def _mix64(z):
    z = (z + 0x9E3779B97F4A7C15) & _MASK
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK
    return z ^ (z >> 31)


def golden_weights(n: int, k: int) -> np.ndarray:
    """Deterministic weight vector k (values in [-1, 1)) for checksums."""
    idx = np.arange(n, dtype=np.uint64)
    z = idx ^ np.uint64((k + 1) << 40)
    z = z + np.uint64(0x9E3779B97F4A7C15)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53 * 2.0 - 1.0


def sample_idx(n: int, count: int = 2048) -> np.ndarray:
    rng = np.random.default_rng(20240607)
    return np.sort(rng.choice(n, size=min(count, n), replace=False))


def summarize(u_steps: np.ndarray) -> dict:
    n = u_steps.shape[1]
    w = [golden_weights(n, k) for k in range(3)]
    return {"norms": np.linalg.norm(u_steps, axis=1),
            "checksums": np.stack([u_steps @ wk for wk in w], axis=1)}


def compare_summary(u_steps, gold, tol):
    """Max relative deviation of norms / checksums (checksums scaled by norm)."""
    s = summarize(u_steps)
    dn = np.max(np.abs(s["norms"] - gold["norms"]) / gold["norms"])
    dc = np.max(np.abs(s["checksums"] - gold["checksums"]) / gold["norms"][:, None])
    return max(dn, dc)
