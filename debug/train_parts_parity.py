"""Config-5 full-size parity (tests/test_gpu_train_cfg5.py) with the training
convs' and the weight gradient's bf16 part counts set: python
debug/train_parts_parity.py CONV_PARTS WGRAD_PARTS"""
import sys
sys.path.insert(0, '.')
from paper_2304_12152_b200 import _lib
_lib.call("ht_set_train_conv_parts", int(sys.argv[1]))
_lib.call("ht_set_wgrad_parts", int(sys.argv[2]))
import pytest
sys.exit(pytest.main(["-q", "-s", "tests/test_gpu_train_cfg5.py", "-p", "no:cacheprovider"]))
