"""Code-matrix uploads above 4M codes are packed on the host (every core,
page-locked buffer) instead of on the device: the packed bytes, the
out-of-range error (the lowest flat index of a code >= k, as k_pack_codes
reports it) and the reference-signature adc_search on host codes
(index.hpp:251-259) are unchanged."""
import numpy as np
import pytest

from oracle import Port
from paper_1908_10396_b200 import anisoq as aq
from paper_1908_10396_b200 import workload as wl

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,M,k", [(90001, 50, 16), (70000, 64, 9), (20000, 230, 200)])
def test_host_packed_upload_round_trip(n, M, k):
    codes = np.random.default_rng(n + M).integers(0, k, (n, M)).astype(np.uint32)
    s = aq.Session.default()
    got = s.upload_codes(aq.CodeMatrix(n, M, k, codes)).download().codes
    assert np.array_equal(got, codes)


def test_host_packed_upload_reports_first_bad_code():
    n, M = 100000, 50
    codes = np.random.default_rng(3).integers(0, 16, (n, M)).astype(np.uint32)
    codes[90000, 1] = 99
    codes[77777, 13] = 16
    with pytest.raises(aq.CodeOutOfRange) as e:
        aq.Session.default().upload_codes(aq.CodeMatrix(n, M, 16, codes))
    assert str(77777 * M + 13) in str(e.value)


def test_dropin_adc_search_on_large_host_codes():
    n, M, k = 120000, 48, 16
    g = np.random.default_rng(9)
    cb = aq.ProductCodebook(M, k, 2, g.standard_normal(M * k * 2) / np.sqrt(2 * M))
    codes = g.integers(0, k, (n, M)).astype(np.uint32)
    q = wl._normalize_rows(g.standard_normal((1, 2 * M)))[0]
    res = aq.adc_search(q, aq.CodeMatrix(n, M, k, codes), cb, 100)
    wi, ws = Port().adc_search_batch(q[None, :], codes, k, cb.dictionaries, M, k, 2, 100)
    assert [h.index for h in res.hits] == wi[0].tolist()
    assert [h.score for h in res.hits] == ws[0].tolist()
