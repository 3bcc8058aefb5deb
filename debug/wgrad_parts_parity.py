import sys; sys.path.insert(0,'.')
from paper_2304_12152_b200 import _lib
parts = int(sys.argv[1])
_lib.call("ht_set_wgrad_parts", parts)
import pytest
sys.exit(pytest.main(["-q", "-s", "tests/test_gpu_train_cfg5.py", "-p", "no:cacheprovider"]))
