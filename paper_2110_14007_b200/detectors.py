"""PyOD-style detector objects over the C ABI (PAPER.md
Appendix D: ``fit`` -> ``decision_scores_`` / ``labels_``,
``decision_function`` for new samples).

Only API plumbing lives here: every score comes from libtod.so (tod_knn,
tod_knn_query, tod_lof, tod_abod); the contamination threshold is the
(1 - contamination) quantile of the training scores (PyOD's convention), taken
on the host from the n fp32 scores the library returns.
"""
from __future__ import annotations

import numpy as np

from .tod import Context


def _host(x):
    return x.cpu().numpy() if hasattr(x, "cpu") else np.asarray(x)


class _Detector:
    def __init__(self, n_neighbors: int = 10, contamination: float = 0.1, device: int = 0,
                 fmt: str = "auto"):
        if not (0.0 < contamination <= 0.5):
            raise ValueError("contamination must be in (0, 0.5]")
        self.n_neighbors = n_neighbors
        self.contamination = contamination
        self.device = device
        self.fmt = fmt
        self._ctx = None

    def _context(self):
        if self._ctx is None:
            self._ctx = Context(device=self.device, fmt=self.fmt)
        return self._ctx

    def _finish_fit(self, scores):
        self.decision_scores_ = _host(scores).astype(np.float64)
        self.threshold_ = float(np.percentile(self.decision_scores_,
                                              100.0 * (1.0 - self.contamination)))
        self.labels_ = (self.decision_scores_ > self.threshold_).astype(np.int64)
        return self

    def predict(self, X=None):
        """Binary labels (1 = outlier) for X, or the training labels if X is None."""
        if X is None:
            return self.labels_
        return (self.decision_function(X) > self.threshold_).astype(np.int64)

    def close(self):
        if self._ctx is not None:
            self._ctx.close()
            self._ctx = None


class KNN(_Detector):
    """kNN outlier detector (Table 1): score = distance to the k-th
    neighbour (``method='largest'``) or the mean kNN distance (``'mean'``)."""

    def __init__(self, n_neighbors: int = 10, method: str = "largest", **kw):
        super().__init__(n_neighbors, **kw)
        if method not in ("largest", "mean"):
            raise ValueError("method must be 'largest' or 'mean'")
        self.method = method

    def fit(self, X):
        self._X = X
        r = self._context().knn(X, self.n_neighbors, want=("score_kth", "score_mean"))
        return self._finish_fit(r.score_kth if self.method == "largest" else r.score_mean)

    def decision_function(self, X):
        r = self._context().knn_query(X, self._X, self.n_neighbors,
                                      want=("score_kth", "score_mean"))
        return _host(r.score_kth if self.method == "largest" else r.score_mean).astype(np.float64)


class LOF(_Detector):
    """Local outlier factor (Breunig 2000) on the exact k-sets."""

    def fit(self, X):
        lof, _, _, _ = self._context().lof(X, self.n_neighbors)
        return self._finish_fit(lof)

    def decision_function(self, X):
        raise NotImplementedError("LOF scores for unseen samples are not part of this build")


class ABOD(_Detector):
    """Angle-based outlier detector (reading A20)."""

    def fit(self, X):
        s, _, _ = self._context().abod(X, self.n_neighbors)
        return self._finish_fit(s)

    def decision_function(self, X):
        raise NotImplementedError("ABOD scores for unseen samples are not part of this build")
