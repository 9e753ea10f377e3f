# idle-poll back-off cap sweep (a DDPMA_BACKOFF knob in a scratch build, 64..4096 ns): no effect on
# timed windows (7.23-7.24e10) nor on e2e (15.2-15.6 s); the knob was not kept.
