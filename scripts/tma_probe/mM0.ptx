.version 8.8
.target sm_100a
.address_size 64
.extern .shared .align 1024 .b8 sm[];
.visible .entry mk(
	.param .align 64 .b8 mk_param_0[128],
	.param .u64 .ptr .align 1 mk_param_1,
	.param .u64 .ptr .align 1 mk_param_2,
	.param .u32 mk_param_3
)
{
	.reg .pred 	%p<9>;
	.reg .b32 	%r<75>;
	.reg .b64 	%rd<20>;
	.reg .f64 	%fd<6>;

	mov.b64 	%rd6, mk_param_0;
	ld.param.u64 	%rd7, [mk_param_2];
	ld.param.u32 	%r32, [mk_param_3];
	cvta.to.global.u64 	%rd1, %rd7;
	mov.u32 	%r74, %tid.x;
	setp.ne.s32 	%p1, %r74, 0;
	@%p1 bra 	$L__BB0_2;
	mov.u32 	%r35, sm;
	add.s32 	%r33, %r35, 9216;
	mov.b32 	%r34, 1;
	// begin inline asm
	mbarrier.init.shared::cta.b64 [%r33], %r34;
	// end inline asm
	// begin inline asm
	fence.mbarrier_init.release.cluster;
	// end inline asm
	// begin inline asm
	fence.proxy.async.shared::cta;
	// end inline asm
$L__BB0_2:
	setp.ne.s32 	%p2, %r74, 0;
	bar.sync 	0;
	@%p2 bra 	$L__BB0_4;
	mov.u32 	%r38, sm;
	add.s32 	%r41, %r38, 9216;
	// begin inline asm
	mbarrier.arrive.expect_tx.shared::cta.b64 _, [%r41], %r32;
	// end inline asm
	cvta.param.u64 	%rd8, %rd6;
	mov.b32 	%r39, 3;
	mov.b32 	%r40, 5;
	// begin inline asm
	cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%r38], [%rd8, {%r39, %r40}], [%r41];
	// end inline asm
$L__BB0_4:
	setp.ne.s32 	%p3, %r74, 0;
	mov.u32 	%r44, sm;
	add.s32 	%r42, %r44, 9216;
	mov.b32 	%r43, 0;
	// begin inline asm
	{
	.reg .pred P1;
W_0:
	mbarrier.try_wait.parity.shared::cta.b64 P1, [%r42], %r43;
	@!P1 bra W_0;
}
	// end inline asm
	bar.sync 	0;
	@%p3 bra 	$L__BB0_6;
	// begin inline asm
	mbarrier.inval.shared::cta.b64 [%r42];
	// end inline asm
$L__BB0_6:
	mov.u32 	%r2, %ntid.x;
	add.s32 	%r47, %r74, %r2;
	max.u32 	%r48, %r47, 1024;
	setp.lt.u32 	%p4, %r47, 1024;
	selp.u32 	%r49, 1, 0, %p4;
	add.s32 	%r50, %r47, %r49;
	sub.s32 	%r51, %r48, %r50;
	div.u32 	%r52, %r51, %r2;
	add.s32 	%r3, %r52, %r49;
	and.b32  	%r53, %r3, 3;
	setp.eq.s32 	%p5, %r53, 3;
	@%p5 bra 	$L__BB0_9;
	add.s32 	%r54, %r3, 1;
	and.b32  	%r55, %r54, 3;
	mul.wide.u32 	%rd10, %r74, 8;
	add.s64 	%rd19, %rd1, %rd10;
	mul.wide.u32 	%rd3, %r2, 8;
	shl.b32 	%r56, %r74, 3;
	add.s32 	%r68, %r44, %r56;
	shl.b32 	%r5, %r2, 3;
	neg.s32 	%r67, %r55;
	mad.lo.s32 	%r74, %r2, %r55, %r74;
$L__BB0_8:
	.pragma "nounroll";
	ld.shared.f64 	%fd1, [%r68];
	st.global.f64 	[%rd19], %fd1;
	add.s64 	%rd19, %rd19, %rd3;
	add.s32 	%r68, %r68, %r5;
	add.s32 	%r67, %r67, 1;
	setp.ne.s32 	%p6, %r67, 0;
	@%p6 bra 	$L__BB0_8;
$L__BB0_9:
	setp.lt.u32 	%p7, %r3, 3;
	@%p7 bra 	$L__BB0_12;
	mad.lo.s32 	%r73, %r2, 3, %r74;
	shl.b32 	%r14, %r2, 2;
	add.s32 	%r58, %r2, %r2;
	add.s32 	%r72, %r74, %r58;
	add.s32 	%r71, %r2, %r74;
	mul.lo.s32 	%r17, %r2, 24;
	shl.b32 	%r59, %r74, 3;
	add.s32 	%r70, %r44, %r59;
	shl.b32 	%r19, %r2, 5;
	shl.b32 	%r20, %r2, 4;
	shl.b32 	%r21, %r2, 3;
$L__BB0_11:
	ld.shared.f64 	%fd2, [%r70];
	mul.wide.u32 	%rd11, %r74, 8;
	add.s64 	%rd12, %rd1, %rd11;
	st.global.f64 	[%rd12], %fd2;
	add.s32 	%r61, %r74, %r2;
	add.s32 	%r62, %r70, %r21;
	ld.shared.f64 	%fd3, [%r62];
	mul.wide.u32 	%rd13, %r71, 8;
	add.s64 	%rd14, %rd1, %rd13;
	st.global.f64 	[%rd14], %fd3;
	add.s32 	%r63, %r61, %r2;
	add.s32 	%r64, %r70, %r20;
	ld.shared.f64 	%fd4, [%r64];
	mul.wide.u32 	%rd15, %r72, 8;
	add.s64 	%rd16, %rd1, %rd15;
	st.global.f64 	[%rd16], %fd4;
	add.s32 	%r65, %r63, %r2;
	add.s32 	%r66, %r70, %r17;
	ld.shared.f64 	%fd5, [%r66];
	mul.wide.u32 	%rd17, %r73, 8;
	add.s64 	%rd18, %rd1, %rd17;
	st.global.f64 	[%rd18], %fd5;
	add.s32 	%r74, %r65, %r2;
	add.s32 	%r73, %r73, %r14;
	add.s32 	%r72, %r72, %r14;
	add.s32 	%r71, %r71, %r14;
	add.s32 	%r70, %r70, %r19;
	setp.lt.u32 	%p8, %r74, 1024;
	@%p8 bra 	$L__BB0_11;
$L__BB0_12:
	ret;

}
