// Experiment (not product code): k_pipe2 <256,256,16,16,2,32,TWT> at 2^16 built with
// experiment macros (-DBFFT_PIPE_NOTW, -DBFFT_PIPE_REDREL, -DBFFT_PIPE_NOFENCE) to price
// each piece; same entry points as exp_wide.cu (table of one config).
#include "exp_wide.cu"
