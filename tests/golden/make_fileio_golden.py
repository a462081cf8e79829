"""Write small FKM1/FKA1 files with the LIVE reference writer (fileio.py:91-152)
so the B200 codec is pinned byte-for-byte even where the reference is absent.

Run in the build container:  python tests/golden/make_fileio_golden.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import flashmeans as fm  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
x32 = fm.generate_dataset(2, 5, 2, 3, 1.0, 7, "single")
fm.write_fkm1(os.path.join(HERE, "ref_small_f32.fkm1"), x32)
x64 = fm.generate_dataset(1, 4, 2, 2, 1.0, 9, "double")
fm.write_fkm1(os.path.join(HERE, "ref_small_f64.fkm1"), x64)
a = fm.Assignments(np.array([[0, 1, 2, 1, 0], [3, 3, 0, 1, 2]], np.int32))
fm.write_fka1(os.path.join(HERE, "ref_small.fka1"), a)
st = fm.AssignmentStore(os.path.join(HERE, "ref_store.fka1"), 2, 5)
st.write_chunk(0, 1, np.array([4, 4], np.int32))
st.write_chunk(1, 3, np.array([1, 2], np.int32))
st.finalize()
np.savez(os.path.join(HERE, "fileio_expected.npz"), x32=x32.data, x64=x64.data, a=a.values)
print("wrote fileio goldens")
