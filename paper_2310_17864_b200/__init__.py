"""B200-native CTC prefix beam-search decoder (ctcb).

Drop-in for the paper's CUDA CTC decoder path (arXiv 2310.17864, PAPER.md:83,
:203) with the reference CPU decoder's exact semantics (ctcforge,
/root/reference/pkg/src/ctcforge/decoder.py:102-817):

    from paper_2310_17864_b200 import cuda_ctc_decoder
    decoder = cuda_ctc_decoder(tokens, nbest=1, beam_size=10, blank_skip_threshold=0.95)
    hyps = decoder(log_probs_cuda_fp32, encoder_out_lens)
"""

from .decoder import (  # noqa: F401
    CUCTCDecoder,
    CUCTCHypothesis,
    DecodeOutput,
    cuda_ctc_decoder,
    skip_cutoff,
)
from .multi import MultiDeviceDecoder  # noqa: F401
from .shard import balanced_ranges, lpt_shards  # noqa: F401
