// common.h — internal helpers shared by the plan layer and the streamer.
#pragma once

int bfft_set_error(int code, const char* fmt, ...);
void bfft_clear_error();
int bfft_last_code();
