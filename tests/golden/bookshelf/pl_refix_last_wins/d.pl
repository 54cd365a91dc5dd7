UCLA pl 1.0

alpha 0 0 : N
beta 4 0 : N
gamma 0 4 : N
delta 5 5 : N
eps 1 7 : N
io_0 9 9 : N /FIXED
ghost 3 3 : N
beta 4.5 0.5 : N
io_0 2 2 : N
alpha 1 1 : N /FIXED
