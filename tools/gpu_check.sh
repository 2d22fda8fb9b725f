ADX_LIB_VARIANT=sktl ADX_ATTN_SK=1 python tools/tools_sk_timeline.py
