#!/bin/bash
# sel_stream_kernel ring geometry on the config-5 shape (segments per tile x stages), all in one
# process per setting list so box drift hits every setting alike (tools/diag_stream_ab.py)
python tools/diag_stream_ab.py 600000000 default SPT=2 SPT=4 SPT=2,ST=3 SPT=8
