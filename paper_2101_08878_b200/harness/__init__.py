"""Application operators of the paper's evaluation on B200s.

* :mod:`.transpose_sum` — ``sum(x + x.T)`` over a chunked fp64 array;
* :mod:`.key_merge` — inner merge of two dataframes on an int64 key.
"""
