"""Concurrent callers (reference contract: pure, concurrency-safe calls,
pkg/README.md:130-131): threads filtering different images through different
paths at the same time get exactly what serial calls give.

Run explicitly (python -m pytest tools/gpu/check_threads.py -m gpu).  The
Python entry points serialise concurrent callers with a process-wide lock
(_lib.serialised); without it (SBF_SERIALISE_CALLS=0) this check, appended
to the whole GPU suite in one process, hit a CUDA illegal memory access in 3
of 6 runs -- see DESIGN.md section 5.  It stays outside the default suite."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import threading

import numpy as np
import pytest

import paper_1203_5128_b200 as P

pytestmark = pytest.mark.gpu


def _cases():
    rng = np.random.default_rng(77)
    out = []
    # K3 sweep (r = 2, 5), split sweep (r = 7, 11), single-pass box, fp64 dual / generic (HDR)
    for shape, ss, sr, kw in [((180, 240), 3.0, 30.0, {}), ((150, 333), 6.0, 20.0, {}),
                              ((200, 210), 8.0, 25.0, {}), ((130, 300), 12.0, 15.0, {}),
                              ((90, 140), 9.0, 30.0, {"spatial": P.Box(9)}),
                              ((96, 128), 4.0, 3000.0, {"hdr": True}), ((70, 90), 2.0, 4000.0, {"hdr": True}),
                              ((64, 200), 6.5, 2500.0, {"hdr": True}),
                              ((80, 100), 2.5, 30.0, {"precision": "hdr"})]:
        hdr = kw.pop("hdr", False)
        img = rng.uniform(0, 65535 if hdr else 255, shape)
        img = np.round(img).astype(np.float32) if hdr else img.astype(np.float32)
        out.append((img, P.FilterParams(sigma_s=ss, sigma_r=sr, epsilon=0.01, **kw)))
    return out


def test_concurrent_threads_match_serial_calls():
    import warnings

    cases = _cases()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        serial = [P.shiftable_bf(img, prm) for img, prm in cases]
        errors, results = [], {}

        def worker(tid):
            try:
                for rep in range(6):
                    for k in range(len(cases)):
                        j = (k + tid) % len(cases)  # every thread walks the paths in a different phase
                        img, prm = cases[j]
                        results[(tid, rep, j)] = P.shiftable_bf(img, prm)
            except Exception as e:  # noqa: BLE001
                errors.append(f"thread {tid}: {type(e).__name__}: {e}")

        threads = [threading.Thread(target=worker, args=(t,)) for t in range(4)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
    assert not errors, errors
    for (tid, rep, j), r in results.items():
        s = serial[j]
        assert (r.plan.T, r.plan.N, r.plan.M) == (s.plan.T, s.plan.N, s.plan.M)
        assert r.fallback_pixels == s.fallback_pixels
        assert np.array_equal(r.image, s.image), (tid, rep, j, float(np.abs(r.image - s.image).max()))


def test_concurrent_threads_on_their_own_streams():
    """The same with one CUDA stream per thread (device tensors in and out):
    kernels of different calls really overlap, so any device-side state shared
    between calls (cached tables, scratch) would show."""
    import warnings

    import torch

    cases = _cases()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        dev = [(torch.from_numpy(img).cuda(), prm) for img, prm in cases]
        serial = [P.shiftable_bf(t, prm) for t, prm in dev]
        torch.cuda.synchronize()
        errors, results = [], {}

        def worker(tid):
            try:
                st = torch.cuda.Stream()
                st.wait_stream(torch.cuda.default_stream())
                with torch.cuda.stream(st):
                    for rep in range(8):
                        for k in range(len(dev)):
                            j = (k + 2 * tid) % len(dev)
                            t, prm = dev[j]
                            results[(tid, rep, j)] = P.shiftable_bf(t, prm)
                st.synchronize()
            except Exception as e:  # noqa: BLE001
                errors.append(f"thread {tid}: {type(e).__name__}: {e}")

        threads = [threading.Thread(target=worker, args=(t,)) for t in range(4)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        torch.cuda.synchronize()
    assert not errors, errors
    for (tid, rep, j), r in results.items():
        s = serial[j]
        assert (r.plan.T, r.plan.N, r.plan.M) == (s.plan.T, s.plan.N, s.plan.M)
        assert torch.equal(r.image, s.image), (tid, rep, j, float((r.image - s.image).abs().max()))
